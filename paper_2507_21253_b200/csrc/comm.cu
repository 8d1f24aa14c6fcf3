// Multi-GPU row sharding: one process per GPU, the handle owns
// an NCCL communicator (NVLink/NVSwitch), B (and A) replicated by broadcast,
// A's rows split by product cost (bsp_partition_rows), each rank multiplies
// its row block with no communication during the multiply, and C stays
// sharded — or is assembled on every rank on request from variable-size
// shards (grouped per-rank broadcasts: NCCL has no all-gather-v; no padding).
// Cluster-wise sharding splits at cluster boundaries (bsp_partition_clusters,
// cluster.cu).
//
// The reference has no distributed code; the split keeps its
// row independence (spgemm.hpp:88-104: rows of C depend only on a row of A
// and on B), so the concatenated shards are C bit for bit.
//
// NCCL is loaded on demand (dlopen of libnccl.so.2, the copy torch already
// mapped when it is in the process), so single-GPU use never needs it.
#include "engine.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>

namespace bsp {
namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl() {
    static NcclApi api{};
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) {
            void* f = dlsym(lib, n);
            if (!f) err = std::string("libnccl lacks ") + n;
            return f;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString =
            reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) throw nccl_error(err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw nccl_error(std::string(what) + ": " + nccl().GetErrorString(r));
}
#define BSP_NCCL(call) ::bsp::nccl_check((call), #call)

ncclComm_t comm_of(bsp_handle h) { return static_cast<ncclComm_t>(h->comm); }

// Rebase the gathered row_ptr: entries [lo, hi) get + off (one launch for all
// ranks' segments: seg_lo/seg_off hold each rank's first row and nnz offset).
__global__ void rebase_rows_kernel(int64_t* __restrict__ rp, int64_t nrows,
                                   const int64_t* __restrict__ seg_lo,
                                   const int64_t* __restrict__ seg_off, int nseg) {
    for (int64_t i = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; i < nrows;
         i += int64_t{gridDim.x} * blockDim.x) {
        // entry i + 1 belongs to the last segment whose first row <= i
        int s = 0;
        while (s + 1 < nseg && seg_lo[s + 1] <= i) ++s;
        rp[i + 1] += seg_off[s];
    }
}

// Elapsed ms between two events recorded on the handle's stream.
struct StreamTimer {
    cudaEvent_t a{}, b{};
    bsp_handle h;
    explicit StreamTimer(bsp_handle hh) : h(hh) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, h->stream);
    }
    double stop() {
        cudaEventRecord(b, h->stream);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    }
    ~StreamTimer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

// Row gather: out row r = A row rows[r] (a warp per output row).
__global__ void select_rows_kernel(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                                   const double* __restrict__ aval, const int32_t* __restrict__ rows,
                                   int64_t n, const int64_t* __restrict__ orp,
                                   int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = int64_t{gridDim.x} * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * int64_t{blockDim.x >> 5} + (threadIdx.x >> 5); r < n; r += nw) {
        const int64_t s = arp[rows[r]], len = arp[rows[r] + 1] - s, d = orp[r];
        for (int64_t q = lane; q < len; q += 32) {
            ocol[d + q] = acol[s + q];
            if (aval) oval[d + q] = aval[s + q];
        }
    }
}
__global__ void select_len_kernel(const int64_t* __restrict__ arp, const int32_t* __restrict__ rows,
                                  int64_t n, int64_t* __restrict__ len) {
    for (int64_t r = blockIdx.x * int64_t{blockDim.x} + threadIdx.x; r < n;
         r += int64_t{gridDim.x} * blockDim.x)
        len[r] = arp[rows[r] + 1] - arp[rows[r]];
}

}  // namespace

// Variable-size all-gather of row shards: rank r holds rows [row_lo_r,
// row_lo_r + nrows_r) as a CSR with row_ptr from 0; every rank receives the
// concatenation in rank order.
void allgather_rows(bsp_handle h, const bsp_csr* shard, bsp_csr* global) {
    const int R = h->comm_size;
    DBuf<int64_t> mine(h, 2), all(h, 2 * R);
    const int64_t mv[2] = {shard->nrows, shard->nnz};
    h2d(h, mine.p, mv, 2);
    BSP_NCCL(nccl().AllGather(mine.p, all.p, 2, ncclInt64, comm_of(h), h->stream));
    std::vector<int64_t> sz(2 * R);
    d2h(h, sz.data(), all.p, 2 * R);
    sync(h);
    std::vector<int64_t> row_lo(R + 1, 0), nnz_off(R + 1, 0);
    for (int r = 0; r < R; ++r) {
        row_lo[r + 1] = row_lo[r] + sz[2 * r];
        nnz_off[r + 1] = nnz_off[r] + sz[2 * r + 1];
    }
    const int64_t n = row_lo[R], nnz = nnz_off[R];
    DBuf<int64_t> rp(h, n + 1, Pool::out);
    ResultPayload pay(h, nnz);
    BSP_CUDA(cudaMemsetAsync(rp.p, 0, sizeof(int64_t), h->stream));
    const int me = h->comm_rank;
    BSP_NCCL(nccl().GroupStart());
    for (int r = 0; r < R; ++r) {
        if (sz[2 * r] > 0)
            BSP_NCCL(nccl().Broadcast(r == me ? shard->row_ptr + 1 : nullptr, rp.p + 1 + row_lo[r],
                                      sz[2 * r], ncclInt64, r, comm_of(h), h->stream));
        if (sz[2 * r + 1] > 0) {
            BSP_NCCL(nccl().Broadcast(r == me ? shard->col_idx : nullptr,
                                      pay.col_idx() + nnz_off[r], sz[2 * r + 1], ncclInt32, r,
                                      comm_of(h), h->stream));
            BSP_NCCL(nccl().Broadcast(r == me ? shard->values : nullptr, pay.values() + nnz_off[r],
                                      sz[2 * r + 1], ncclFloat64, r, comm_of(h), h->stream));
        }
    }
    BSP_NCCL(nccl().GroupEnd());
    if (n > 0) {
        DBuf<int64_t> seg(h, 2 * R);
        h2d(h, seg.p, row_lo.data(), R);
        h2d(h, seg.p + R, nnz_off.data(), R);
        const unsigned grid =
            static_cast<unsigned>(std::min<int64_t>(div_up(n, 256), int64_t{h->sm_count} * 8));
        BSP_LAUNCH(h, rebase_rows_kernel, grid, 256, 0, rp.p, n, seg.p, seg.p + R, R);
    }
    global->nrows = n;
    global->ncols = shard->ncols;
    global->nnz = nnz;
    global->row_ptr = rp.release();
    global->col_idx = pay.col_idx();
    global->values = pay.block.release();
    global->owned = 2;
}

}  // namespace bsp

using namespace bsp;

extern "C" {

int bsp_nccl_unique_id(void* id_out) {
    return guarded([&] {
        require(id_out != nullptr, "nccl_unique_id: null out");
        static_assert(sizeof(ncclUniqueId) == BSP_NCCL_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        BSP_NCCL(nccl().GetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int bsp_comm_init(bsp_handle h, int nranks, int rank, const void* id) {
    return guarded([&] {
        require(h != nullptr && id != nullptr, "comm_init: null argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad rank / nranks");
        require(h->comm == nullptr, "comm_init: the handle already has a communicator");
        BSP_CUDA(cudaSetDevice(h->device));
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        ncclComm_t c = nullptr;
        BSP_NCCL(nccl().CommInitRank(&c, nranks, uid, rank));
        h->comm = c;
        h->comm_rank = rank;
        h->comm_size = nranks;
    });
}

int bsp_comm_destroy(bsp_handle h) {
    return guarded([&] {
        if (!h || !h->comm) return;
        BSP_CUDA(cudaStreamSynchronize(h->stream));
        BSP_NCCL(nccl().CommDestroy(comm_of(h)));
        h->comm = nullptr;
        h->comm_rank = 0;
        h->comm_size = 1;
    });
}

int bsp_comm_rank(bsp_handle h, int* rank, int* nranks) {
    return guarded([&] {
        require(h != nullptr, "comm_rank: null handle");
        if (rank) *rank = h->comm_rank;
        if (nranks) *nranks = h->comm_size;
    });
}

int bsp_csr_broadcast(bsp_handle h, bsp_csr* M, int root, double* ms_out) {
    return guarded([&] {
        require(M != nullptr, "csr_broadcast: null matrix");
        require(root >= 0 && root < h->comm_size, "csr_broadcast: bad root");
        BSP_CUDA(cudaSetDevice(h->device));
        StreamTimer tm(h);
        if (h->comm_size == 1) {
            if (ms_out) *ms_out = tm.stop();
            return;
        }
        DBuf<int64_t> shp(h, 3);
        if (h->comm_rank == root) {
            check_csr(M, "csr_broadcast");
            const int64_t v[3] = {M->nrows, M->ncols, M->nnz};
            h2d(h, shp.p, v, 3);
        }
        BSP_NCCL(nccl().Broadcast(shp.p, shp.p, 3, ncclInt64, root, comm_of(h), h->stream));
        int64_t v[3];
        d2h(h, v, shp.p, 3);
        sync(h);
        if (h->comm_rank != root) {
            M->nrows = v[0];
            M->ncols = v[1];
            M->nnz = v[2];
            DBuf<int64_t> rp(h, v[0] + 1, Pool::out);
            DBuf<int32_t> ci(h, v[2], Pool::out);
            DBuf<double> va(h, v[2], Pool::out);
            M->row_ptr = rp.release();
            M->col_idx = ci.release();
            M->values = va.release();
            M->owned = 1;
        }
        BSP_NCCL(nccl().GroupStart());
        BSP_NCCL(nccl().Broadcast(M->row_ptr, M->row_ptr, v[0] + 1, ncclInt64, root, comm_of(h),
                                  h->stream));
        if (v[2] > 0) {
            BSP_NCCL(nccl().Broadcast(M->col_idx, M->col_idx, v[2], ncclInt32, root, comm_of(h),
                                      h->stream));
            BSP_NCCL(nccl().Broadcast(M->values, M->values, v[2], ncclFloat64, root, comm_of(h),
                                      h->stream));
        }
        BSP_NCCL(nccl().GroupEnd());
        const double ms = tm.stop();
        if (ms_out) *ms_out = ms;
    });
}

int bsp_csr_allgather_rows(bsp_handle h, const bsp_csr* shard, bsp_csr* global) {
    return guarded([&] {
        require(shard != nullptr && global != nullptr, "csr_allgather_rows: null argument");
        BSP_CUDA(cudaSetDevice(h->device));
        if (h->comm_size == 1 || h->comm == nullptr) {
            // one rank: the shard is the global C (a copy, so ownership stays simple)
            DBuf<int64_t> rp(h, shard->nrows + 1, Pool::out);
            ResultPayload pay(h, shard->nnz);
            BSP_CUDA(cudaMemcpyAsync(rp.p, shard->row_ptr, (shard->nrows + 1) * sizeof(int64_t),
                                     cudaMemcpyDeviceToDevice, h->stream));
            if (shard->nnz > 0) {
                BSP_CUDA(cudaMemcpyAsync(pay.col_idx(), shard->col_idx, shard->nnz * sizeof(int32_t),
                                         cudaMemcpyDeviceToDevice, h->stream));
                BSP_CUDA(cudaMemcpyAsync(pay.values(), shard->values, shard->nnz * sizeof(double),
                                         cudaMemcpyDeviceToDevice, h->stream));
            }
            *global = bsp_csr{shard->nrows, shard->ncols, shard->nnz, rp.release(), pay.col_idx(),
                              pay.values(), 2};
            pay.block.release();
            return;
        }
        allgather_rows(h, shard, global);
    });
}

// Rows `rows` (device int32, any order, repeats allowed) of A as a new CSR:
// the operand of a cluster shard (the rows of its clusters, in cluster order).
int bsp_csr_select_rows(bsp_handle h, const bsp_csr* A, const int32_t* rows, int64_t n,
                        bsp_csr* out) {
    return guarded([&] {
        check_csr(A, "csr_select_rows");
        require(out != nullptr && (rows != nullptr || n == 0), "csr_select_rows: null argument");
        BSP_CUDA(cudaSetDevice(h->device));
        DBuf<int64_t> len(h, n + 1), rp(h, n + 1, Pool::out);
        BSP_CUDA(cudaMemsetAsync(len.p, 0, (n + 1) * sizeof(int64_t), h->stream));
        const unsigned g1 = static_cast<unsigned>(
            std::max<int64_t>(1, std::min<int64_t>(div_up(n, 256), int64_t{h->sm_count} * 8)));
        if (n > 0) BSP_LAUNCH(h, select_len_kernel, g1, 256, 0, A->row_ptr, rows, n, len.p);
        exclusive_scan_i64(h, len.p, rp.p, n + 1);
        const int64_t nnz = read_scalar(h, rp.p + n);
        DBuf<int32_t> ci(h, nnz, Pool::out);
        DBuf<double> va(h, nnz, Pool::out);
        const unsigned g2 = static_cast<unsigned>(
            std::max<int64_t>(1, std::min<int64_t>(div_up(n, 8), int64_t{h->sm_count} * 16)));
        if (n > 0)
            BSP_LAUNCH(h, select_rows_kernel, g2, 256, 0, A->row_ptr, A->col_idx, A->values, rows, n,
                       rp.p, ci.p, A->values ? va.p : nullptr);
        *out = bsp_csr{n, A->ncols, nnz, rp.release(), ci.release(), va.release(), 1};
    });
}

// SPMD: every rank calls it with A and B resident (bsp_csr_broadcast them
// first).  The split is computed identically on every rank from A and B.
int bsp_spgemm_rowwise_sharded(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int gather,
                               bsp_csr* C, bsp_shard_info* info) {
    return guarded([&] {
        require(C != nullptr, "spgemm_rowwise_sharded: null output");
        check_csr(A, "spgemm_rowwise_sharded");
        check_csr(B, "spgemm_rowwise_sharded");
        BSP_CUDA(cudaSetDevice(h->device));
        const int R = h->comm_size, me = h->comm_rank;
        auto check = [](int rc) {
            if (rc != BSP_OK) throw std::runtime_error(bsp_last_error());
        };
        const void* key[4] = {A->row_ptr, A->col_idx, B->row_ptr, B->col_idx};
        const bool cached = static_cast<int>(h->part_bounds.size()) == R + 1 &&
                            std::equal(key, key + 4, h->part_key) && h->part_nnz[0] == A->nnz &&
                            h->part_nnz[1] == B->nnz;
        if (!cached) {
            h->part_bounds.assign(R + 1, 0);
            check(bsp_partition_rows(h, A, B, R, h->part_bounds.data()));
            std::copy(key, key + 4, h->part_key);
            h->part_nnz[0] = A->nnz;
            h->part_nnz[1] = B->nnz;
        }
        const std::vector<int64_t>& bounds = h->part_bounds;
        const int64_t r0 = bounds[me], r1 = bounds[me + 1];
        bsp_shard_info inf{};
        inf.row_begin = r0;
        inf.row_end = r1;
        StreamTimer tm(h);
        bsp_csr shard{};
        rowwise_multiply(h, A, B, r0, r1, &shard, nullptr, nullptr);
        inf.multiply_ms = tm.stop();
        inf.products_local = h->stats.products;
        inf.nnz_local = shard.nnz;
        if (gather && R > 1) {
            StreamTimer tg(h);
            try {
                allgather_rows(h, &shard, C);
            } catch (...) {
                bsp_csr_free(h, &shard);
                throw;
            }
            inf.gather_ms = tg.stop();
            bsp_csr_free(h, &shard);
            inf.nnz_global = C->nnz;
        } else {
            *C = shard;
            inf.nnz_global = R == 1 ? shard.nnz : -1;
        }
        if (info) *info = inf;
    });
}

}  // extern "C"
