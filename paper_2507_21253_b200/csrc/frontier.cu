// Tall-skinny frontier operands on the device: batched BFS.
//
// Replaces reference generate_frontiers (frontier.hpp:20-77), the B side of
// the paper's square x tall-skinny workload (bench.hpp:145-151): `width =
// min(batch, n)` sources (sorted prefix of a seeded shuffle, :37-46), one BFS
// per source over A's rows as out-neighbour lists (:48-63), and frontier t =
// the n x width 0/1 matrix {(v, s) : depth_s(v) == t} (:65-76), at most
// num_frontiers of them.
//
// All sources advance together, level-synchronously: the level-t frontier is
// a list of (source, vertex) pairs; one warp per pair walks the vertex's row
// and claims unvisited (source, neighbour) cells of the depth table with
// atomicCAS (-1 -> t+1) — each cell is claimed exactly once, so the depth of
// every (s, v) equals the reference's sequential BFS depth whatever the claim
// order.  Frontier t is then built as CSR from its pair list (count, scan,
// scatter, per-row sort of the source columns), so it is identical to the
// reference's (rows ascending, columns ascending, values 1.0).
#include "engine.cuh"

#include <algorithm>
#include <memory>
#include <vector>

namespace bsp {

std::vector<int32_t> random_permutation(int64_t n, uint64_t seed);  // host_reorder.cpp

namespace {

__device__ __forceinline__ uint64_t pack_pair(int32_t s, int32_t v) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(s)) << 32) | static_cast<uint32_t>(v);
}

__global__ void bfs_seed_kernel(const int32_t* __restrict__ sources, int64_t width, int64_t n,
                                int32_t* __restrict__ depth, uint64_t* __restrict__ cur) {
    const int64_t s = blockIdx.x * int64_t{blockDim.x} + threadIdx.x;
    if (s >= width) return;
    depth[s * n + sources[s]] = 0;
    cur[s] = pack_pair(static_cast<int32_t>(s), sources[s]);
}

// Out-degree sum of the frontier's vertices: capacity bound of the next level.
__global__ void frontier_degree_kernel(const int64_t* __restrict__ rp,
                                       const uint64_t* __restrict__ cur, int64_t ncur,
                                       int64_t* __restrict__ deg) {
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < ncur;
         i += int64_t{gridDim.x} * blockDim.x) {
        const int32_t v = static_cast<int32_t>(cur[i] & 0xffffffffu);
        deg[i] = rp[v + 1] - rp[v];
    }
}

// One warp per (source, vertex) pair of level t: claim unvisited neighbours.
__global__ void bfs_expand_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  int64_t n, const uint64_t* __restrict__ cur, int64_t ncur,
                                  int32_t* __restrict__ depth, int32_t next_level,
                                  uint64_t* __restrict__ next,
                                  unsigned long long* __restrict__ next_cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t{gridDim.x} * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * int64_t{blockDim.x} + threadIdx.x) >> 5; i < ncur; i += warps) {
        const uint64_t pr = cur[i];
        const int32_t s = static_cast<int32_t>(pr >> 32);
        const int32_t v = static_cast<int32_t>(pr & 0xffffffffu);
        int32_t* d = depth + static_cast<int64_t>(s) * n;
        const int64_t e0 = rp[v], e1 = rp[v + 1];
        for (int64_t e = e0; e < e1; e += 32) {
            bool won = false;
            int32_t w = 0;
            if (e + lane < e1) {
                w = __ldg(ci + e + lane);
                won = atomicCAS(d + w, -1, next_level) == -1;
            }
            const unsigned m = __ballot_sync(0xffffffffu, won);
            if (m == 0) continue;
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(next_cnt, static_cast<unsigned long long>(__popc(m)));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (won) next[base + __popc(m & ((1u << lane) - 1u))] = pack_pair(s, w);
        }
    }
}

__global__ void frontier_count_kernel(const uint64_t* __restrict__ cur, int64_t ncur,
                                      int64_t* __restrict__ rowcnt) {
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < ncur;
         i += int64_t{gridDim.x} * blockDim.x)
        atomicAdd(reinterpret_cast<unsigned long long*>(
                      &rowcnt[static_cast<int32_t>(cur[i] & 0xffffffffu)]), 1ull);
}

__global__ void frontier_scatter_kernel(const uint64_t* __restrict__ cur, int64_t ncur,
                                        int64_t* __restrict__ cursor, int32_t* __restrict__ col) {
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < ncur;
         i += int64_t{gridDim.x} * blockDim.x) {
        const int32_t v = static_cast<int32_t>(cur[i] & 0xffffffffu);
        const int64_t pos =
            static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long*>(&cursor[v]), 1ull));
        col[pos] = static_cast<int32_t>(cur[i] >> 32);
    }
}

// Rows hold at most `width` sources (a handful on average): insertion sort.
__global__ void frontier_sort_kernel(const int64_t* __restrict__ rp, int64_t n,
                                     int32_t* __restrict__ col, double* __restrict__ val) {
    for (int64_t r = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; r < n;
         r += int64_t{gridDim.x} * blockDim.x) {
        const int64_t b = rp[r], e = rp[r + 1];
        for (int64_t p = b + 1; p < e; ++p) {
            const int32_t k = col[p];
            int64_t q = p - 1;
            while (q >= b && col[q] > k) {
                col[q + 1] = col[q];
                --q;
            }
            col[q + 1] = k;
        }
        for (int64_t p = b; p < e; ++p) val[p] = 1.0;
    }
}

int grid_of(bsp_handle h, int64_t items, int block) {
    return static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(div_up(std::max<int64_t>(items, 1), block), int64_t{h->sm_count} * 16)));
}

// Frontier pair list -> n x width CSR (output pool, owned = 2).
void frontier_to_csr(bsp_handle h, const uint64_t* cur, int64_t ncur, int64_t n, int64_t width,
                     bsp_csr* out) {
    DBuf<int64_t> cnt(h, n + 1);
    BSP_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(int64_t), h->stream));
    BSP_LAUNCH(h, frontier_count_kernel, grid_of(h, ncur, 256), 256, 0, cur, ncur, cnt.p);
    DBuf<int64_t> rp(h, n + 1, Pool::out);
    exclusive_scan_i64(h, cnt.p, rp.p, n + 1);
    BSP_CUDA(cudaMemcpyAsync(cnt.p, rp.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                             h->stream));
    ResultPayload pay(h, ncur);
    BSP_LAUNCH(h, frontier_scatter_kernel, grid_of(h, ncur, 256), 256, 0, cur, ncur, cnt.p,
               pay.col_idx());
    BSP_LAUNCH(h, frontier_sort_kernel, grid_of(h, n, 256), 256, 0, rp.p, n, pay.col_idx(),
               pay.values());
    out->nrows = n;
    out->ncols = width;
    out->nnz = ncur;
    out->row_ptr = rp.release();
    out->col_idx = pay.col_idx();
    out->values = pay.block.release();
    out->owned = 2;
}

// Frontiers made so far; released unless handed to the caller.
struct FrontierList {
    bsp_handle h;
    std::unique_ptr<bsp_csr[]> items;
    int64_t n = 0;
    FrontierList(bsp_handle hh, int64_t cap) : h(hh), items(new bsp_csr[cap]) {}
    ~FrontierList() {
        for (int64_t i = 0; i < n; ++i) bsp_csr_free(h, &items[i]);
    }
};

void generate_frontiers(bsp_handle h, const bsp_csr* A, int64_t num_frontiers, int64_t batch,
                        uint64_t seed, bsp_csr* out, int64_t* count) {
    *count = 0;
    const int64_t n = A->nrows;
    if (n == 0) return;
    const int64_t width = std::min(batch, n);
    // sources: sorted prefix of the seeded shuffle (frontier.hpp:37-46)
    std::vector<int32_t> src = random_permutation(n, seed);
    src.resize(static_cast<size_t>(width));
    std::sort(src.begin(), src.end());
    DBuf<int32_t> dsrc(h, width);
    h2d(h, dsrc.p, src.data(), width);
    DBuf<int32_t> depth(h, width * n);
    BSP_CUDA(cudaMemsetAsync(depth.p, 0xff, static_cast<size_t>(width * n) * sizeof(int32_t),
                             h->stream));
    DBuf<uint64_t> cur(h, width);
    BSP_LAUNCH(h, bfs_seed_kernel, grid_of(h, width, 128), 128, 0, dsrc.p, width, n, depth.p,
               cur.p);
    int64_t ncur = width;
    FrontierList made(h, num_frontiers);
    for (int32_t t = 0;; ++t) {
        bsp_csr f{};
        frontier_to_csr(h, cur.p, ncur, n, width, &f);
        made.items[made.n++] = f;
        if (made.n == num_frontiers) break;
        // next level: capacity = out-degree sum of this frontier
        DBuf<int64_t> deg(h, ncur);
        BSP_LAUNCH(h, frontier_degree_kernel, grid_of(h, ncur, 256), 256, 0, A->row_ptr, cur.p,
                   ncur, deg.p);
        const int64_t cap = std::min(reduce_sum_i64(h, deg.p, ncur), width * n);
        if (cap == 0) break;
        DBuf<uint64_t> next(h, cap);
        DBuf<unsigned long long> nc(h, 1);
        BSP_CUDA(cudaMemsetAsync(nc.p, 0, sizeof(unsigned long long), h->stream));
        BSP_LAUNCH(h, bfs_expand_kernel, grid_of(h, ncur * 32, 256), 256, 0, A->row_ptr,
                   A->col_idx, n, cur.p, ncur, depth.p, t + 1, next.p, nc.p);
        const int64_t nn = static_cast<int64_t>(read_scalar(h, nc.p));
        if (nn == 0) break;  // every search has exhausted its component
        cur = std::move(next);
        ncur = nn;
    }
    for (int64_t t = 0; t < made.n; ++t) out[t] = made.items[t];
    *count = made.n;
    made.n = 0;  // ownership passed to the caller
}

}  // namespace

}  // namespace bsp

using namespace bsp;

extern "C" {

int bsp_generate_frontiers(bsp_handle h, const bsp_csr* A, int64_t num_frontiers, int64_t batch,
                           uint64_t seed, bsp_csr* out, int64_t* count) {
    return guarded([&] {
        require(h && out && count, "generate_frontiers: null argument");
        check_csr(A, "generate_frontiers");
        require(A->nrows == A->ncols, "generate_frontiers: adjacency must be square");
        require(num_frontiers >= 1, "generate_frontiers: num_frontiers must be >= 1");
        require(batch >= 1, "generate_frontiers: batch must be >= 1");
        BSP_CUDA(cudaSetDevice(h->device));
        generate_frontiers(h, A, num_frontiers, batch, seed, out, count);
    });
}

}  // extern "C"
