// Candidate-pair generation for hierarchical clustering on sm_100a.
//
// (1) bsp_spgemm_topk replaces reference spgemm_topk (spgemm.hpp:144-206):
//     the binarized A*A^T overlap counts are produced by the same ESC tiles as
//     the row-wise product (count = length of a run of equal columns, exact),
//     converted to Jaccard o/(n_i+n_j-o) with one IEEE double division, and a
//     per-row top-k by (score desc, j asc) is selected on chip.  Heavy rows
//     select per window and merge.  The reference's serial unordered-pair
//     dedup (first emitter in ascending i wins) is reproduced exactly as a
//     parallel rule: (i,j) from row i is dropped iff j < i and i is in row j's
//     kept list.  The output list is therefore element-for-element identical.
// (2) bsp_minhash_candidates: north-star item (4), not in the reference
//     (PAPER.md:555-565 replaced LSH by top-k): 32-bit minhash signatures,
//     LSH banding by radix sort of band keys, bucket-local pairs, exact
//     Jaccard verification, per-row top-k with the same order and dedup rule.
#include "esc.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include <algorithm>

namespace bsp {

namespace {

constexpr int MAXTOPK = 32;

// Warp-level selection of the best `topk` (score desc, j asc) among n
// candidates stored in (sc, jj); selected entries are marked with -1.
__device__ int warp_select_topk(double* sc, uint32_t* jj, int n, int topk, int32_t* oj,
                                double* os) {
    const int lane = threadIdx.x & 31;
    int got = 0;
    for (int r = 0; r < topk; ++r) {
        double bs = -1.0;
        uint32_t bj = 0xffffffffu;
        int bi = -1;
        for (int e = lane; e < n; e += 32) {
            const double s = sc[e];
            const uint32_t j = jj[e];
            if (s >= 0.0 && (s > bs || (s == bs && j < bj))) {
                bs = s;
                bj = j;
                bi = e;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double s2 = __shfl_xor_sync(0xffffffffu, bs, o);
            const uint32_t j2 = __shfl_xor_sync(0xffffffffu, bj, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (s2 > bs || (s2 == bs && j2 < bj)) {
                bs = s2;
                bj = j2;
                bi = i2;
            }
        }
        if (bi < 0) break;
        if (lane == 0) {
            oj[r] = static_cast<int32_t>(bj);
            os[r] = bs;
            sc[bi] = -1.0;
        }
        __syncwarp();
        ++got;
    }
    return got;
}

template <int T, int I>
__global__ void __launch_bounds__(T) topk_tile_kernel(Mats m, const int32_t* __restrict__ ids,
                                                      const Window* __restrict__ wins, int topk,
                                                      double th, int32_t* __restrict__ rj,
                                                      double* __restrict__ rs,
                                                      int32_t* __restrict__ rn,
                                                      int32_t* __restrict__ wj,
                                                      double* __restrict__ ws,
                                                      int32_t* __restrict__ wn) {
    using S = EscShared<T, I, true>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& s = *reinterpret_cast<S*>(smem_raw);
    __shared__ int s_nc;
    const int tid = threadIdx.x;
    const int32_t id = ids[blockIdx.x];
    int32_t row, c0, c1, w = -1;
    int64_t wsofs = -1;
    int wwi = 0;
    if (wins) {
        w = id;
        const Window wd = wins[w];
        row = wd.row;
        c0 = wd.c0;
        c1 = wd.c1;
        wsofs = wd.sofs;
        wwi = wd.wi;
    } else {
        row = id;
        c0 = 0;
        c1 = m.ncols;
    }
    if (tid == 0) s_nc = 0;
    const int total = expand_products<T, I, false>(m, row, c0, c1, wins == nullptr, s, wsofs, wwi);
    const uint32_t width = static_cast<uint32_t>(c1 - c0);
    const int bits = bit_length(width);
    uint32_t k[I], v[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const int e = tid * I + i;
        k[i] = e < total ? s.keys[e] : width;
        v[i] = static_cast<uint32_t>(e);
    }
    __syncthreads();
    typename S::Sort(s.u.sort).Sort(k, v, 0, bits);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < I; ++i) s.keys[tid * I + i] = k[i];
    __syncthreads();
    const double ni = static_cast<double>(m.arp[row + 1] - m.arp[row]);
#pragma unroll
    for (int i = 0; i < I; ++i) {
        const int e0 = tid * I + i;
        if (e0 < total && (e0 == 0 || s.keys[e0 - 1] != k[i])) {
            int e = e0 + 1;
            while (e < total && s.keys[e] == k[i]) ++e;
            const int32_t j = static_cast<int32_t>(k[i]) + c0;
            if (j != row) {
                // reference spgemm.hpp:174-177: o / (nnz_i + nnz_j - o), doubles
                const double o = static_cast<double>(e - e0);
                const double nj = static_cast<double>(m.arp[j + 1] - m.arp[j]);
                const double score = o / (ni + nj - o);
                if (score >= th) {
                    const int idx = atomicAdd(&s_nc, 1);
                    s.vals[idx] = score;
                    s.u.sidx[idx] = static_cast<uint32_t>(j);
                }
            }
        }
    }
    __syncthreads();
    if (tid < 32) {
        const int nc = s_nc;
        int32_t* oj = w >= 0 ? wj + int64_t{w} * topk : rj + int64_t{row} * topk;
        double* os = w >= 0 ? ws + int64_t{w} * topk : rs + int64_t{row} * topk;
        const int got = warp_select_topk(s.vals, s.u.sidx, nc, topk, oj, os);
        if (tid == 0) (w >= 0 ? wn[w] : rn[row]) = got;
    }
}

// Streaming warp top-k over `count` candidates produced by get(e) -> (score, j):
// batches of up to 224 candidates are merged with the running best list.
constexpr int STREAM_BUF = 256;

template <typename Get>
__device__ int warp_topk_stream(Get get, int64_t count, int topk, double* buf_s, uint32_t* buf_j,
                                int32_t* best_j, double* best_s) {
    const int lane = threadIdx.x & 31;
    int nb = 0;
    int64_t cur = 0;
    do {
        for (int t = lane; t < nb; t += 32) {
            buf_s[t] = best_s[t];
            buf_j[t] = static_cast<uint32_t>(best_j[t]);
        }
        const int64_t left = count - cur;
        const int64_t take = left < (STREAM_BUF - MAXTOPK) ? left : (STREAM_BUF - MAXTOPK);
        for (int64_t t = lane; t < take; t += 32) {
            double sc;
            uint32_t jj;
            get(cur + t, sc, jj);
            buf_s[nb + t] = sc;
            buf_j[nb + t] = jj;
        }
        __syncwarp();
        cur += take;
        nb = warp_select_topk(buf_s, buf_j, nb + static_cast<int>(take), topk, best_j, best_s);
        __syncwarp();
    } while (cur < count);
    return nb;
}

// Heavy rows: merge the per-window lists of a row (windows of one row are
// contiguous; the row's first window carries the merge).
__global__ void topk_merge_windows_kernel(const Window* __restrict__ wins, int64_t nwin, int topk,
                                          const int32_t* __restrict__ wj,
                                          const double* __restrict__ ws,
                                          const int32_t* __restrict__ wn,
                                          const int64_t* __restrict__ wcand_off,
                                          int32_t* __restrict__ rj, double* __restrict__ rs,
                                          int32_t* __restrict__ rn) {
    __shared__ double bs[8][STREAM_BUF];
    __shared__ uint32_t bj[8][STREAM_BUF];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t w = (blockIdx.x * int64_t{blockDim.x} + threadIdx.x) >> 5;
    if (w >= nwin || wins[w].first != w) return;
    const int32_t row = wins[w].row;
    int64_t we = w + 1;
    while (we < nwin && wins[we].first == w) ++we;
    // candidates of windows [w, we) are the entries ws/wj[v*topk + t], t < wn[v];
    // enumerate them through the exclusive offsets wcand_off.
    const int64_t base = wcand_off[w];
    const int64_t count = wcand_off[we] - base;
    auto get = [&](int64_t e, double& sc, uint32_t& jj) {
        // locate window v with wcand_off[v] <= base+e < wcand_off[v+1]
        int64_t lo = w, hi = we - 1;
        const int64_t x = base + e;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (wcand_off[mid] <= x) lo = mid; else hi = mid - 1;
        }
        const int64_t t = x - wcand_off[lo];
        sc = ws[lo * topk + t];
        jj = static_cast<uint32_t>(wj[lo * topk + t]);
    };
    const int got = warp_topk_stream(get, count, topk, bs[wib], bj[wib], rj + int64_t{row} * topk,
                                     rs + int64_t{row} * topk);
    if (lane == 0) rn[row] = got;
}

// Reference dedup (spgemm.hpp:193-204) as a parallel rule.
__global__ void topk_dedup_kernel(int64_t n, int topk, const int32_t* __restrict__ rj,
                                  const int32_t* __restrict__ rn, uint8_t* __restrict__ keep,
                                  int32_t* __restrict__ kept_cnt) {
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < n;
         i += int64_t{gridDim.x} * blockDim.x) {
        int kc = 0;
        for (int t = 0; t < rn[i]; ++t) {
            const int32_t j = rj[i * topk + t];
            bool dup = false;
            if (j < i)
                for (int u = 0; u < rn[j]; ++u)
                    if (rj[int64_t{j} * topk + u] == i) dup = true;
            keep[i * topk + t] = dup ? 0 : 1;
            kc += dup ? 0 : 1;
        }
        kept_cnt[i] = kc;
    }
}

__global__ void topk_emit_kernel(int64_t n, int topk, const int32_t* __restrict__ rj,
                                 const double* __restrict__ rs, const int32_t* __restrict__ rn,
                                 const uint8_t* __restrict__ keep, const int64_t* __restrict__ off,
                                 bsp_candidate* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < n;
         i += int64_t{gridDim.x} * blockDim.x) {
        int64_t o = off[i];
        for (int t = 0; t < rn[i]; ++t) {
            if (!keep[i * topk + t]) continue;
            out[o].i = static_cast<int32_t>(i);
            out[o].j = rj[i * topk + t];
            out[o].score = rs[i * topk + t];
            ++o;
        }
    }
}

template <int T, int I>
void launch_topk(bsp_handle h, const Mats& m, const int32_t* ids, int64_t n, const Window* wins,
                 int topk, double th, int32_t* rj, double* rs, int32_t* rn, int32_t* wj, double* ws,
                 int32_t* wn) {
    if (n <= 0) return;
    using S = EscShared<T, I, true>;
    auto k = topk_tile_kernel<T, I>;
    static const std::string nm = "topk_tile<" + std::to_string(T) + "x" + std::to_string(I) + ">";
    set_smem(k, sizeof(S));
    BSP_LAUNCH_AS(h, nm.c_str(), k, static_cast<unsigned>(n), T, sizeof(S), m, ids, wins, topk, th, rj, rs, rn,
               wj, ws, wn);
}

int grid_of(bsp_handle h, int64_t n, int block) {
    return static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(div_up(std::max<int64_t>(n, 1), block), int64_t{h->sm_count} * 16)));
}

// Per-row candidate lists (rj/rs/rn, topk slots per row) -> reference-order
// deduplicated host list.
void emit_candidates(bsp_handle h, int64_t n, int topk, const int32_t* rj, const double* rs,
                     const int32_t* rn, bsp_candidate** pairs_out, int64_t* npairs_out) {
    DBuf<uint8_t> keep(h, n * topk);
    DBuf<int32_t> kc(h, n + 1);
    BSP_CUDA(cudaMemsetAsync(kc.p, 0, (n + 1) * sizeof(int32_t), h->stream));
    BSP_LAUNCH(h, topk_dedup_kernel, grid_of(h, n, 256), 256, 0, n, topk, rj, rn, keep.p, kc.p);
    DBuf<int64_t> off(h, n + 1);
    exclusive_scan_i32_to_i64(h, kc.p, off.p, n + 1);
    const int64_t np = read_scalar(h, off.p + n);
    DBuf<bsp_candidate> out(h, np);
    BSP_LAUNCH(h, topk_emit_kernel, grid_of(h, n, 256), 256, 0, n, topk, rj, rs, rn, keep.p, off.p,
               out.p);
    bsp_candidate* host = host_malloc<bsp_candidate>(np);
    d2h(h, host, out.p, np);
    sync(h);
    *pairs_out = host;
    *npairs_out = np;
}

// ---------------------------------------------------------------------------
// minhash / LSH
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t hash32(uint32_t x, uint64_t seed) {
    uint64_t z = (static_cast<uint64_t>(x) << 1 | 1ull) * 0x9E3779B97F4A7C15ull ^ seed;
    z ^= z >> 31;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 29;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 32;
    return static_cast<uint32_t>(z);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}

// One warp per row: nhash minimum hashes of the row's column set.
__global__ void minhash_sig_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                   int64_t n, int nhash, uint64_t seed, uint32_t* __restrict__ sig) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t{blockDim.x} + threadIdx.x) >> 5;
    const int64_t nw = (int64_t{gridDim.x} * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nw) {
        const int64_t b = rp[i], e = rp[i + 1];
        for (int hh = lane; hh < nhash; hh += 32) {
            const uint64_t hs = mix64(seed + 0x9E3779B97F4A7C15ull * (hh + 1));
            uint32_t mn = 0xffffffffu;
            for (int64_t p = b; p < e; ++p) mn = min(mn, hash32(static_cast<uint32_t>(col[p]), hs));
            sig[i * nhash + hh] = mn;
        }
    }
}

__global__ void band_keys_kernel(const int64_t* __restrict__ rp, const uint32_t* __restrict__ sig,
                                 int64_t n, int nhash, int bands, uint64_t* __restrict__ keys,
                                 int32_t* __restrict__ vals) {
    const int r = nhash / bands;
    for (int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; t < n * bands;
         t += int64_t{gridDim.x} * blockDim.x) {
        const int64_t i = t % n;
        const int b = static_cast<int>(t / n);
        uint64_t k = mix64(0x1234567ull + b);
        for (int q = 0; q < r; ++q) k = mix64(k ^ sig[i * nhash + b * r + q]);
        if (rp[i + 1] == rp[i]) k = ~0ull;  // empty rows never collide
        keys[t] = k == ~0ull && rp[i + 1] != rp[i] ? k - 1 : k;
        vals[t] = static_cast<int32_t>(i);
    }
}

// Bucket-local pairs: each sorted element pairs with the next `win` members
// of its bucket (all pairs for buckets of size <= win+1).
template <int MODE>
__global__ void lsh_pairs_kernel(const uint64_t* __restrict__ keys, const int32_t* __restrict__ rows,
                                 int64_t m, int win, int32_t* __restrict__ cnt,
                                 const int64_t* __restrict__ off, uint64_t* __restrict__ pairs) {
    for (int64_t e = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; e < m;
         e += int64_t{gridDim.x} * blockDim.x) {
        int c = 0;
        const uint64_t k = keys[e];
        if (k != ~0ull) {
            for (int d = 1; d <= win && e + d < m && keys[e + d] == k; ++d) {
                if (MODE) {
                    const uint32_t a = static_cast<uint32_t>(rows[e]), b = static_cast<uint32_t>(rows[e + d]);
                    const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
                    pairs[off[e] + c] = (static_cast<uint64_t>(lo) << 32) | hi;
                }
                ++c;
            }
        }
        if (!MODE) cnt[e] = c;
    }
}

// Exact Jaccard of each unique pair; writes directed entries (i->j and j->i)
// with key (i<<32|j) when score >= th.
__global__ void verify_pairs_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                    const uint64_t* __restrict__ pairs, int64_t np, double th,
                                    uint64_t* __restrict__ dkeys, double* __restrict__ dscore) {
    for (int64_t t = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; t < np;
         t += int64_t{gridDim.x} * blockDim.x) {
        const uint64_t pr = pairs[t];
        const int64_t i = static_cast<int64_t>(pr >> 32), j = static_cast<int64_t>(pr & 0xffffffffu);
        int64_t p = rp[i], q = rp[j], inter = 0;
        const int64_t pe = rp[i + 1], qe = rp[j + 1];
        while (p < pe && q < qe) {
            const int32_t a = col[p], b = col[q];
            inter += (a == b);
            p += (a <= b);
            q += (b <= a);
        }
        const int64_t uni = (pe - rp[i]) + (qe - rp[j]) - inter;
        const double s = uni == 0 ? 0.0 : static_cast<double>(inter) / static_cast<double>(uni);
        const bool ok = (i != j) && s >= th;
        dkeys[2 * t] = ok ? ((static_cast<uint64_t>(i) << 32) | static_cast<uint64_t>(j)) : ~0ull;
        dkeys[2 * t + 1] = ok ? ((static_cast<uint64_t>(j) << 32) | static_cast<uint64_t>(i)) : ~0ull;
        dscore[2 * t] = s;
        dscore[2 * t + 1] = s;
    }
}

// Directed entries sorted by (i, j): per row select topk by (score desc, j asc).
__global__ void rows_topk_kernel(const uint64_t* __restrict__ dkeys, const double* __restrict__ ds,
                                 int64_t m, int64_t n, int topk, int32_t* __restrict__ rj,
                                 double* __restrict__ rs, int32_t* __restrict__ rn) {
    __shared__ double bs[8][STREAM_BUF];
    __shared__ uint32_t bj[8][STREAM_BUF];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warp = (blockIdx.x * int64_t{blockDim.x} + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t{gridDim.x} * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nwarps) {
        auto lb = [&](uint64_t key) {
            int64_t lo = 0, hi = m;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (dkeys[mid] < key) lo = mid + 1; else hi = mid;
            }
            return lo;
        };
        const int64_t b = lb(static_cast<uint64_t>(i) << 32);
        const int64_t e = lb(static_cast<uint64_t>(i + 1) << 32);
        auto get = [&](int64_t t, double& sc, uint32_t& jj) {
            sc = ds[b + t];
            jj = static_cast<uint32_t>(dkeys[b + t] & 0xffffffffu);
        };
        const int got = warp_topk_stream(get, e - b, topk, bs[wib], bj[wib], rj + i * topk,
                                         rs + i * topk);
        if (lane == 0) rn[i] = got;
        __syncwarp();
    }
}

// Dense heavy windows of A*A^T: per-column overlap counters in smem.
constexpr int TDT = 256;
struct TopkDenseShared {
    int32_t cnt[WD];
    double cs[WD];
    uint32_t cj[WD];
    int nc;
};

__global__ void __launch_bounds__(TDT) topk_dense_kernel(Mats m, const int32_t* __restrict__ ids,
                                                         const Window* __restrict__ wins, int topk,
                                                         double th, int32_t* __restrict__ wj,
                                                         double* __restrict__ ws,
                                                         int32_t* __restrict__ wn) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TopkDenseShared& s = *reinterpret_cast<TopkDenseShared*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t w = ids[blockIdx.x];
    const Window wd = wins[w];
    const int32_t row = wd.row, c0 = wd.c0, c1 = wd.c1;
    for (int e = tid; e < WD; e += TDT) s.cnt[e] = 0;
    if (tid == 0) s.nc = 0;
    __syncthreads();
    for (int64_t p = m.arp[row] + warp; p < m.arp[row + 1]; p += TDT / 32) {
        int64_t b0, b1;
        segment_range(m, false, wd.sofs, wd.wi, p, m.arp[row], m.arp[row + 1] - m.arp[row], c0,
                      c1, b0, b1);
        for (int64_t q = b0 + lane; q < b1; q += 32) atomicAdd(&s.cnt[__ldg(m.bcol + q) - c0], 1);
    }
    __syncthreads();
    const double ni = static_cast<double>(m.arp[row + 1] - m.arp[row]);
    for (int e = tid; e < WD; e += TDT) {
        const int32_t j = c0 + e;
        if (j >= c1 || s.cnt[e] == 0 || j == row) continue;
        const double o = static_cast<double>(s.cnt[e]);
        const double nj = static_cast<double>(m.arp[j + 1] - m.arp[j]);
        const double score = o / (ni + nj - o);
        if (score >= th) {
            const int idx = atomicAdd(&s.nc, 1);
            s.cs[idx] = score;
            s.cj[idx] = static_cast<uint32_t>(j);
        }
    }
    __syncthreads();
    if (tid < 32) {
        const int got = warp_select_topk(s.cs, s.cj, s.nc, topk, wj + int64_t{w} * topk,
                                         ws + int64_t{w} * topk);
        if (tid == 0) wn[w] = got;
    }
}

}  // namespace

}  // namespace bsp

using namespace bsp;

extern "C" {

int bsp_spgemm_topk(bsp_handle h, const bsp_csr* A, const bsp_csr* At, int32_t topk,
                    double jacc_th, bsp_candidate** pairs_out, int64_t* npairs_out) {
    return guarded([&] {
        check_csr(A, "spgemm_topk");
        check_csr(At, "spgemm_topk");
        require(A->ncols == At->nrows, "spgemm_topk: dimension mismatch");
        require(topk >= 1, "spgemm_topk: topk must be >= 1");
        require(topk <= MAXTOPK, "spgemm_topk: topk > 32 not supported on the device");
        require(pairs_out && npairs_out, "spgemm_topk: null output");
        BSP_CUDA(cudaSetDevice(h->device));
        const int64_t n = A->nrows;
        const Mats m = make_mats(A, At);
        RowwisePlan plan;
        build_plan(h, m, 0, n, nullptr, plan, nullptr);
        DBuf<int32_t> rj(h, n * topk), rn(h, n + 1);
        DBuf<double> rs(h, n * topk);
        BSP_CUDA(cudaMemsetAsync(rn.p, 0, (n + 1) * sizeof(int32_t), h->stream));
        DBuf<int32_t> wj(h, plan.nwin * topk), wn(h, plan.nwin + 1);
        DBuf<double> ws(h, plan.nwin * topk);
        BSP_CUDA(cudaMemsetAsync(wn.p, 0, (plan.nwin + 1) * sizeof(int32_t), h->stream));
        const int64_t* co = plan.class_off;
        const int64_t* cc = plan.class_count;
        launch_topk<32, 4>(h, m, plan.lists.p + co[1], cc[1], nullptr, topk, jacc_th, rj.p, rs.p,
                           rn.p, wj.p, ws.p, wn.p);
        launch_topk<64, 8>(h, m, plan.lists.p + co[2], cc[2], nullptr, topk, jacc_th, rj.p, rs.p,
                           rn.p, wj.p, ws.p, wn.p);
        // light classes 3 and 4 (<= 1024, <= 2048 products) share the
        // 2048-product tile, classes 5 and 6 (<= 3072, <= 4096) the 4096 one
        // (adjacent in the row list)
        static_assert(NCLS == 8, "top-k launches one tile per light class pair");
        launch_topk<128, 16>(h, m, plan.lists.p + co[3], cc[3] + cc[4], nullptr, topk, jacc_th,
                             rj.p, rs.p, rn.p, wj.p, ws.p, wn.p);
        launch_topk<256, 16>(h, m, plan.lists.p + co[5], cc[5] + cc[6], nullptr, topk, jacc_th,
                             rj.p, rs.p, rn.p, wj.p, ws.p, wn.p);
        if (plan.nwin > 0) {
            const Mats mw = plan.with_starts(m);
            launch_topk<256, 16>(h, mw, plan.sparse_ids.p, plan.nsparse, plan.wins.p, topk, jacc_th,
                                 rj.p, rs.p, rn.p, wj.p, ws.p, wn.p);
            set_smem(topk_dense_kernel, sizeof(TopkDenseShared));
            BSP_LAUNCH(h, topk_dense_kernel, static_cast<unsigned>(plan.ndense), TDT,
                       sizeof(TopkDenseShared), mw,
                       plan.dense_ids.p, plan.wins.p, topk, jacc_th, wj.p, ws.p, wn.p);
            DBuf<int64_t> woff(h, plan.nwin + 1);
            exclusive_scan_i32_to_i64(h, wn.p, woff.p, plan.nwin + 1);
            BSP_LAUNCH(h, topk_merge_windows_kernel,
                       static_cast<unsigned>(div_up(plan.nwin * 32, 256)), 256, 0, plan.wins.p,
                       plan.nwin, topk, wj.p, ws.p, wn.p, woff.p, rj.p, rs.p, rn.p);
        }
        emit_candidates(h, n, topk, rj.p, rs.p, rn.p, pairs_out, npairs_out);
    });
}

int bsp_minhash_candidates(bsp_handle h, const bsp_csr* A, int32_t nhash, int32_t bands,
                           uint64_t seed, int32_t topk, double jacc_th, bsp_candidate** pairs_out,
                           int64_t* npairs_out) {
    return guarded([&] {
        check_csr(A, "minhash_candidates");
        require(nhash >= 1 && bands >= 1 && nhash % bands == 0,
                "minhash_candidates: nhash must be a positive multiple of bands");
        require(topk >= 1 && topk <= MAXTOPK, "minhash_candidates: topk must be in [1, 32]");
        BSP_CUDA(cudaSetDevice(h->device));
        const int64_t n = A->nrows;
        DBuf<uint32_t> sig(h, n * nhash);
        BSP_LAUNCH(h, minhash_sig_kernel, grid_of(h, n * 32, 256), 256, 0, A->row_ptr, A->col_idx, n,
                   nhash, seed, sig.p);
        const int64_t m = n * bands;
        DBuf<uint64_t> keys(h, m), keys2(h, m);
        DBuf<int32_t> vals(h, m), vals2(h, m);
        BSP_LAUNCH(h, band_keys_kernel, grid_of(h, m, 256), 256, 0, A->row_ptr, sig.p, n, nhash,
                   bands, keys.p, vals.p);
        size_t tmp = 0;
        BSP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, keys2.p, vals.p, vals2.p, m,
                                                 0, 64, h->stream));
        {
            DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
            BSP_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, keys.p, keys2.p, vals.p, vals2.p, m,
                                                     0, 64, h->stream));
            ++h->launches;
        }
        const int win = 8;
        DBuf<int32_t> cnt(h, m + 1);
        BSP_CUDA(cudaMemsetAsync(cnt.p, 0, (m + 1) * sizeof(int32_t), h->stream));
        BSP_LAUNCH(h, lsh_pairs_kernel<0>, grid_of(h, m, 256), 256, 0, keys2.p, vals2.p, m, win,
                   cnt.p, nullptr, nullptr);
        DBuf<int64_t> off(h, m + 1);
        exclusive_scan_i32_to_i64(h, cnt.p, off.p, m + 1);
        const int64_t np = read_scalar(h, off.p + m);
        DBuf<uint64_t> pairs(h, np), pairs2(h, np);
        BSP_LAUNCH(h, lsh_pairs_kernel<1>, grid_of(h, m, 256), 256, 0, keys2.p, vals2.p, m, win,
                   nullptr, off.p, pairs.p);
        // unique pairs
        tmp = 0;
        BSP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, pairs.p, pairs2.p, np, 0, 64,
                                                h->stream));
        int64_t nu = 0;
        DBuf<uint64_t> upairs(h, np);
        {
            DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
            BSP_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, pairs.p, pairs2.p, np, 0, 64,
                                                    h->stream));
            DBuf<int64_t> nrun(h, 1);
            DBuf<int32_t> lens(h, np);
            size_t tmp2 = 0;
            BSP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp2, pairs2.p, upairs.p, lens.p,
                                                        nrun.p, np, h->stream));
            DBuf<uint8_t> t2(h, static_cast<int64_t>(tmp2));
            BSP_CUDA(cub::DeviceRunLengthEncode::Encode(t2.p, tmp2, pairs2.p, upairs.p, lens.p,
                                                        nrun.p, np, h->stream));
            h->launches += 2;
            nu = read_scalar(h, nrun.p);
        }
        DBuf<uint64_t> dkeys(h, 2 * nu), dkeys2(h, 2 * nu);
        DBuf<double> dsc(h, 2 * nu), dsc2(h, 2 * nu);
        BSP_LAUNCH(h, verify_pairs_kernel, grid_of(h, nu, 256), 256, 0, A->row_ptr, A->col_idx,
                   upairs.p, nu, jacc_th, dkeys.p, dsc.p);
        tmp = 0;
        BSP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dkeys.p, dkeys2.p, dsc.p, dsc2.p,
                                                 2 * nu, 0, 64, h->stream));
        {
            DBuf<uint8_t> t(h, static_cast<int64_t>(tmp));
            BSP_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, dkeys.p, dkeys2.p, dsc.p, dsc2.p,
                                                     2 * nu, 0, 64, h->stream));
            ++h->launches;
        }
        DBuf<int32_t> rj(h, n * topk), rn(h, n + 1);
        DBuf<double> rs(h, n * topk);
        BSP_CUDA(cudaMemsetAsync(rn.p, 0, (n + 1) * sizeof(int32_t), h->stream));
        BSP_LAUNCH(h, rows_topk_kernel, grid_of(h, n * 32, 256), 256, 0, dkeys2.p, dsc2.p, 2 * nu, n,
                   topk, rj.p, rs.p, rn.p);
        emit_candidates(h, n, topk, rj.p, rs.p, rn.p, pairs_out, npairs_out);
    });
}

}  // extern "C"
