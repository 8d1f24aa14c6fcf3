/*
 * bsp.h — C ABI of the B200-native cluster-wise SpGEMM engine.
 *
 * This is the drop-in boundary for the reference's header-only C++ API in
 * namespace cspgemm (reference: proj/include/cspgemm/cspgemm.hpp:1-16).
 * Every entry point below names the reference function it replaces
 * (file:line under /root/reference/proj/include/cspgemm/).
 *
 * Conventions
 *  - All functions return BSP_OK (0) or a BSP_ERR_* code; no exception ever
 *    crosses the ABI.  BSP_ERR_CONTRACT corresponds to the reference's
 *    cspgemm::contract_error (types.hpp:16-19); BSP_ERR_IO to io_error
 *    (types.hpp:23-26).  bsp_last_error() returns the message of the last
 *    failure on the calling thread.
 *  - Device matrices (bsp_csr, bsp_csr_cluster) hold DEVICE pointers.
 *    Row offsets are int64 (the reference's int32 index_t, types.hpp:11,
 *    overflows for nnz(C) > 2^31-1); column indices are int32; values f64.
 *  - Host matrices (bsp_host_csr) hold HOST pointers (malloc'ed by the
 *    library when returned; release with bsp_host_csr_free).
 *  - All device work is stream-ordered on the handle's stream.  A handle is
 *    used by one host thread at a time; distinct handles are independent.
 *  - Buffers the library allocates for results are released with
 *    bsp_csr_free / bsp_csr_cluster_free.
 */
#ifndef BSP_H_
#define BSP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSP_OK 0
#define BSP_ERR_CONTRACT 1
#define BSP_ERR_OOM 2
#define BSP_ERR_CUDA 3
#define BSP_ERR_NCCL 4
#define BSP_ERR_IO 5
#define BSP_ERR_INTERNAL 6

typedef struct bsp_handle_s* bsp_handle;

/* Device CSR.  reference: CsrMatrix, csr.hpp:51-88 (int64 row_ptr here). */
typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t* row_ptr; /* device, nrows+1 */
    int32_t* col_idx; /* device, nnz */
    double* values;   /* device, nnz */
    int32_t owned;    /* 0: caller's arrays; 1: library-allocated (released by
                         bsp_csr_free); 2: library-allocated, col_idx shares the
                         values block (results of a multiply) */
} bsp_csr;

/* Host CSR (library- or caller-owned host memory). */
typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t* row_ptr;
    int32_t* col_idx;
    double* values;
} bsp_host_csr;

/* Device CSR_Cluster.  reference: CsrClusterMatrix, cluster_format.hpp:94-125.
 * value slot of (cluster c, merged column position p, member l) is
 * value_ptr[c] + p*cluster_sizes[c] + l; valid bit per slot (uint64 words);
 * member_mask[cluster_col_ptr[c] + p] has bit l set iff that slot is valid
 * (derived from valid; used by the cluster kernel; cluster sizes <= 32).
 * csr_* is a device CSR copy of the rows (original row order) kept for the
 * clusters the engine routes to the row-wise bins (singletons, heavy). */
typedef struct {
    int64_t nclusters, nrows, ncols;
    int64_t ncolslots; /* cluster_col_ptr[nclusters] */
    int64_t nslots;    /* value_ptr[nclusters] */
    int32_t* cluster_sizes;   /* [nclusters] */
    int64_t* member_ptr;      /* [nclusters+1] offsets into row_map */
    int64_t* cluster_col_ptr; /* [nclusters+1] */
    int32_t* col_idx;         /* [ncolslots] */
    int64_t* value_ptr;       /* [nclusters+1] */
    double* values;           /* [nslots] */
    uint64_t* valid;          /* [(nslots+63)/64] */
    uint32_t* member_mask;    /* [ncolslots] */
    int32_t* row_map;         /* [nrows] */
    int64_t* csr_row_ptr;     /* [nrows+1] row view (may be NULL) */
    int32_t* csr_col_idx;
    double* csr_values;
    int32_t owned;
    int64_t csr_nnz;          /* nnz of the row view (0: unknown / no view) */
} bsp_csr_cluster;

/* Host mirror of CSR_Cluster (for download / host-side checks). */
typedef struct {
    int64_t nclusters, nrows, ncols, ncolslots, nslots;
    int32_t* cluster_sizes;
    int64_t* cluster_col_ptr;
    int32_t* col_idx;
    int64_t* value_ptr;
    double* values;
    uint64_t* valid;
    int32_t* row_map;
} bsp_host_csr_cluster;

/* reference: AccessStats, cluster_spgemm.hpp:26-30 */
typedef struct {
    uint64_t b_row_loads;
    uint64_t a_inner_iters;
    uint64_t placeholder_skips;
} bsp_access_stats;

/* reference: CandidatePair, spgemm.hpp:132-136 */
typedef struct {
    int32_t i, j;
    double score;
} bsp_candidate;

/* Per-call execution statistics of the row-wise / cluster-wise engine. */
typedef struct {
    int64_t products;     /* sum over rows of intermediate products */
    int64_t nnz_out;      /* nnz(C) */
    int64_t units[16];    /* work units: [0..7] rows per class (0 empty; 1..6 light, at
                             most 128/512/1024/2048/3072/4096 products; 7 heavy), [8]
                             sparse windows, [9] dense windows, [10] cluster tiles, [11]
                             of which union tiles (each B entry sorted once per cluster),
                             [12] two-row clusters on the cluster hash accumulator, [13]
                             rows of duplicate-heavy clusters whose B-row reuse is too low
                             to pay, run on the row-wise hash accumulator, [14] device
                             allocations the call had to ask the driver for (0 once a
                             repeated multiply is served from the handle's block cache) */
    int32_t kernels_launched;
    int32_t chunks;       /* row chunks: bsp_spgemm_rowwise_host splits A's rows when C
                             exceeds the device budget (half the free memory); 1 otherwise */
} bsp_exec_stats;

/* ------------------------------------------------------------------ */
/* handle / memory                                                     */
/* ------------------------------------------------------------------ */
const char* bsp_last_error(void);
const char* bsp_version(void);
int bsp_create(int device, bsp_handle* out);
int bsp_destroy(bsp_handle h);
/* Run on an external stream (e.g. torch's current stream); NULL = the legacy
 * default stream. */
int bsp_set_stream(bsp_handle h, void* cuda_stream);
/* Per-launch CUDA-event profiling of engine kernels (bench / diagnostics).
 * bsp_profile_report synchronises, writes "name\tlaunches\tms\n" lines into
 * buf (NUL-terminated, truncated to cap) and returns the full length. */
int bsp_profile(bsp_handle h, int on);
int64_t bsp_profile_report(bsp_handle h, char* buf, int64_t cap);
void* bsp_get_stream(bsp_handle h);
int bsp_synchronize(bsp_handle h);
/* Number of engine kernels launched by this handle since creation. */
int64_t bsp_kernel_launches(bsp_handle h);
int bsp_get_exec_stats(bsp_handle h, bsp_exec_stats* out);

/* Upload a host CSR (int64 or int32 row offsets) into library-owned device memory. */
int bsp_csr_upload(bsp_handle h, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                   const int32_t* col_idx, const double* values, bsp_csr* out);
int bsp_csr_upload_rp32(bsp_handle h, int64_t nrows, int64_t ncols, const int32_t* row_ptr,
                        const int32_t* col_idx, const double* values, bsp_csr* out);
/* Wrap caller-owned device arrays (not freed by bsp_csr_free). */
int bsp_csr_view(int64_t nrows, int64_t ncols, int64_t nnz, int64_t* row_ptr,
                 int32_t* col_idx, double* values, bsp_csr* out);
/* Copy a device CSR into caller-provided host arrays (sizes from the struct). */
int bsp_csr_download(bsp_handle h, const bsp_csr* m, int64_t* row_ptr, int32_t* col_idx,
                     double* values);
/* Same, enqueued on the handle's stream without synchronising. */
int bsp_csr_download_async(bsp_handle h, const bsp_csr* m, int64_t* row_ptr, int32_t* col_idx,
                           double* values);
/* Make `waiter`'s stream wait for all work enqueued so far on `signaler`'s. */
int bsp_stream_wait(bsp_handle waiter, bsp_handle signaler);
int bsp_csr_free(bsp_handle h, bsp_csr* m);
/* Pinned host allocation helpers (for end-to-end host-buffer calls). */
int bsp_host_alloc(size_t bytes, void** out);
int bsp_host_free(void* p);

/* ------------------------------------------------------------------ */
/* row-wise SpGEMM (the hot path)                                      */
/* ------------------------------------------------------------------ */
/* Per-row intermediate products (device int64 [nrows]) and their total.
 * reference: detail::row_upper_bound, spgemm.hpp:31-36 */
int bsp_spgemm_products(bsp_handle h, const bsp_csr* A, const bsp_csr* B,
                        int64_t* row_products_dev, int64_t* total_out);
/* Exact per-row output counts (device int64 [nrows]).
 * reference: spgemm_symbolic, spgemm.hpp:41-63 */
int bsp_spgemm_symbolic(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int64_t* counts_dev);
/* C = A*B, rows sorted, structural zeros kept, every value accumulated as
 * ((0 + a_i,k1*b_k1,j) + a_i,k2*b_k2,j) + ... in ascending k with separately
 * rounded multiply and add (bit-identical to the reference).
 * reference: spgemm_rowwise, spgemm.hpp:70-106 */
int bsp_spgemm_rowwise(bsp_handle h, const bsp_csr* A, const bsp_csr* B, bsp_csr* C);
/* Same product restricted to A rows [row_begin, row_end) (a row shard);
 * C has row_end-row_begin rows. */
int bsp_spgemm_rowwise_range(bsp_handle h, const bsp_csr* A, const bsp_csr* B,
                             int64_t row_begin, int64_t row_end, bsp_csr* C);
/* Host-buffer entry point mirroring the reference's value-returning call:
 * uploads A and B, multiplies, returns C in library-malloc'ed host arrays
 * (bsp_host_csr_free).  B may alias A (A*A). */
int bsp_spgemm_rowwise_host(bsp_handle h, const bsp_host_csr* A, const bsp_host_csr* B,
                            bsp_host_csr* C);
/* Balanced contiguous row split of A by cumulative intermediate products
 * (SURVEY 8(e)); bounds_out has nparts+1 entries (host). */
int bsp_partition_rows(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int32_t nparts,
                       int64_t* bounds_out);

/* ------------------------------------------------------------------ */
/* multi-GPU (one process per GPU; NCCL over NVLink, loaded on demand)  */
/* ------------------------------------------------------------------ */
/* No reference counterpart: the reference has no distributed code
 * (SPEC.md:563).  Rows of C are independent given B (spgemm.hpp:88-104), so
 * A's rows are split by product cost (bsp_partition_rows), B is replicated,
 * and each rank multiplies its row block with no communication; C stays
 * sharded or is assembled on request. */
#define BSP_NCCL_ID_BYTES 128
typedef struct {
    int64_t row_begin, row_end; /* this rank's rows of A (and of C) */
    int64_t products_local;     /* intermediate products of this rank's rows */
    int64_t nnz_local;          /* nnz of this rank's shard of C */
    int64_t nnz_global;         /* nnz of the gathered C (gather=1 or one rank), else -1 */
    double multiply_ms;         /* this rank's multiply (CUDA events, handle stream) */
    double gather_ms;           /* the assembly of the global C (gather=1) */
} bsp_shard_info;
/* An ncclUniqueId (rank 0 creates it and ships it to the others, e.g. with
 * torch.distributed). */
int bsp_nccl_unique_id(void* id_out /* BSP_NCCL_ID_BYTES */);
/* Give the handle its own NCCL communicator (on its device). */
int bsp_comm_init(bsp_handle h, int nranks, int rank, const void* id /* BSP_NCCL_ID_BYTES */);
int bsp_comm_destroy(bsp_handle h);
int bsp_comm_rank(bsp_handle h, int* rank, int* nranks);
/* Replicate a device CSR from `root` to every rank (NCCL broadcasts on the
 * handle's stream; on the other ranks M is allocated by the library, owned=1).
 * ms_out (nullable): the broadcast's time (CUDA events). */
int bsp_csr_broadcast(bsp_handle h, bsp_csr* M, int root, double* ms_out);
/* Global C from row shards held by every rank (concatenated in rank order):
 * an all-gather of the shard sizes, then one broadcast per rank of its exact
 * arrays (no padding; NCCL has no all-gather-v) and a row_ptr rebase. */
int bsp_csr_allgather_rows(bsp_handle h, const bsp_csr* shard, bsp_csr* global);
/* Row-sharded C = A*B: this rank's row block of C (gather = 0) or the global C
 * on every rank (gather = 1).  A and B must be resident on every rank. */
int bsp_spgemm_rowwise_sharded(bsp_handle h, const bsp_csr* A, const bsp_csr* B, int gather,
                               bsp_csr* C, bsp_shard_info* info /* nullable */);
/* Cluster-wise shards: bounds[0..nparts] over clusters (CSR_Cluster order),
 * split by the clusters' intermediate products, snapped to cluster boundaries. */
int bsp_partition_clusters(bsp_handle h, const bsp_csr_cluster* A, const bsp_csr* B,
                           int32_t nparts, int64_t* bounds_out);
/* Rows `rows` (device int32) of A as a new CSR (owned): a cluster shard's
 * operand (its clusters' rows in cluster order). */
int bsp_csr_select_rows(bsp_handle h, const bsp_csr* A, const int32_t* rows, int64_t n,
                        bsp_csr* out);

/* ------------------------------------------------------------------ */
/* cluster-wise SpGEMM                                                 */
/* ------------------------------------------------------------------ */
/* reference: build_csr_cluster, cluster_format.hpp:130-186.  cluster_ptr/rows
 * are the flattened ClusterAssignment (host arrays). */
int bsp_csr_cluster_build(bsp_handle h, const bsp_csr* A, int64_t nclusters,
                          const int64_t* cluster_ptr, const int32_t* rows,
                          bsp_csr_cluster* out);
int bsp_csr_cluster_free(bsp_handle h, bsp_csr_cluster* m);
int bsp_csr_cluster_download(bsp_handle h, const bsp_csr_cluster* m, bsp_host_csr_cluster* out);
void bsp_host_csr_cluster_free(bsp_host_csr_cluster* m);
/* C = A*B with A clustered; C written directly as CSR over the original row
 * indices (bit-identical to bsp_spgemm_rowwise on cluster_to_csr(A)).  When
 * C_cluster is non-NULL the CSR_Cluster form of C is produced as well
 * (reference: spgemm_clusterwise, cluster_spgemm.hpp:186-189). */
int bsp_spgemm_clusterwise(bsp_handle h, const bsp_csr_cluster* A, const bsp_csr* B,
                           bsp_csr* C, bsp_csr_cluster* C_cluster);
/* reference: cluster_to_csr, cluster_format.hpp:190-233 */
int bsp_cluster_to_csr(bsp_handle h, const bsp_csr_cluster* m, bsp_csr* out);
/* reference: AccessStats of spgemm_clusterwise_instrumented (cluster_spgemm.hpp:191-197)
 * and rowwise_access_stats (:34-45) — counting kernels outside the timed path. */
int bsp_cluster_access_stats(bsp_handle h, const bsp_csr_cluster* A, const bsp_csr* B,
                             bsp_access_stats* out);
int bsp_rowwise_access_stats(bsp_handle h, const bsp_csr* A, const bsp_csr* B,
                             bsp_access_stats* out);

/* ------------------------------------------------------------------ */
/* clustering / candidate generation                                   */
/* ------------------------------------------------------------------ */
/* Device transpose (rows of the result sorted).  reference: transpose, csr.hpp:115-135 */
int bsp_transpose(bsp_handle h, const bsp_csr* A, bsp_csr* out);
/* Tall-skinny frontier operands by batched BFS on the device.  reference:
 * generate_frontiers, frontier.hpp:20-77 (identical matrices: sources = sorted
 * prefix of reorder_random(n, seed), frontier t = {(v, s): depth_s(v) == t}).
 * `out` must hold num_frontiers entries; *count receives how many were made
 * (fewer when every search exhausts its component).  Each is n x min(batch, n),
 * library-owned (bsp_csr_free). */
int bsp_generate_frontiers(bsp_handle h, const bsp_csr* A, int64_t num_frontiers, int64_t batch,
                           uint64_t seed, bsp_csr* out, int64_t* count);
/* reference: spgemm_topk, spgemm.hpp:144-206 (element-for-element identical
 * output list, scores bitwise).  Results in library-malloc'ed host memory
 * (free with bsp_host_free_plain). a/a_t patterns only (values ignored). */
int bsp_spgemm_topk(bsp_handle h, const bsp_csr* A, const bsp_csr* At, int32_t topk,
                    double jacc_th, bsp_candidate** pairs_out, int64_t* npairs_out);
/* Minhash/LSH candidate generation (north-star item 4; not in the reference):
 * nhash signatures per row, `bands` LSH bands, candidates verified by exact
 * Jaccard >= jacc_th, at most topk per row kept with the reference's
 * (score desc, j asc) order and dedup rule. */
int bsp_minhash_candidates(bsp_handle h, const bsp_csr* A, int32_t nhash, int32_t bands,
                           uint64_t seed, int32_t topk, double jacc_th,
                           bsp_candidate** pairs_out, int64_t* npairs_out);
/* Hierarchical clustering: GPU candidates + host heap/union-find merge.
 * reference: hierarchical_clusters, clustering.hpp:109-185.  method 0 = top-k
 * (pinned to the reference), 1 = minhash (nhash/bands used).  Output is the
 * flattened assignment: cluster_ptr [nclusters+1], rows [nrows] (malloc'ed). */
int bsp_hierarchical_clusters(bsp_handle h, const bsp_host_csr* A, double jacc_th,
                              int32_t max_cluster, int32_t method, int32_t nhash,
                              int32_t bands, uint64_t seed, int64_t* nclusters_out,
                              int64_t** cluster_ptr_out, int32_t** rows_out);
/* Host merge only, from an external candidate list (reference clustering.hpp:122-183). */
int bsp_merge_candidates(const bsp_host_csr* A, const bsp_candidate* pairs, int64_t npairs,
                         double jacc_th, int32_t max_cluster, int64_t* nclusters_out,
                         int64_t** cluster_ptr_out, int32_t** rows_out,
                         int64_t* nmerges_out, bsp_candidate** merges_out);
/* reference: variable_length_clusters (clustering.hpp:76-93), fixed_length (:59-69) */
int bsp_variable_length_clusters(const bsp_host_csr* A, double jacc_th, int32_t max_cluster,
                                 int64_t* nclusters_out, int64_t** cluster_ptr_out,
                                 int32_t** rows_out);
int bsp_fixed_length_clusters(int64_t nrows, int32_t k, int64_t* nclusters_out,
                              int64_t** cluster_ptr_out, int32_t** rows_out);
/* reference: jaccard_similarity, spgemm.hpp:110-129 */
int bsp_jaccard(const bsp_host_csr* A, int64_t i, int64_t j, double* out);

/* ------------------------------------------------------------------ */
/* host preprocessing (reference reorder.hpp / csr.hpp)                */
/* ------------------------------------------------------------------ */
/* perm[new] = old.  reference: reorder_random (reorder.hpp:20-30) */
int bsp_reorder_random(int64_t n, uint64_t seed, int32_t* perm_out);
/* reference: reorder_rcm (reorder.hpp:137-181) — permutation-identical */
int bsp_reorder_rcm(const bsp_host_csr* A, int32_t* perm_out);
/* reference: reorder_degree (reorder.hpp:33-40) */
int bsp_reorder_degree(const bsp_host_csr* A, int32_t* perm_out);
/* reference: bandwidth (reorder.hpp:44-51) */
int bsp_bandwidth(const bsp_host_csr* A, int64_t* out);
/* reference: permute_symmetric (csr.hpp:146-172), permute_rows (:175-193) */
int bsp_permute_symmetric(const bsp_host_csr* A, const int32_t* perm, bsp_host_csr* out);
int bsp_permute_rows(const bsp_host_csr* A, const int32_t* perm, bsp_host_csr* out);
/* reference: transpose (csr.hpp:115-135), host form */
int bsp_transpose_host(const bsp_host_csr* A, bsp_host_csr* out);
void bsp_host_csr_free(bsp_host_csr* m);

/* ------------------------------------------------------------------ */
/* file IO (host; reference matrix_market.hpp)                          */
/* ------------------------------------------------------------------ */
/* load_matrix_market (matrix_market.hpp:42-119) + coo_to_csr (csr.hpp:92-113):
 * coordinate real/integer/pattern, general/symmetric; 1-based -> 0-based;
 * symmetric files expanded; duplicates summed; BSP_ERR_IO "path:line: msg". */
int bsp_load_matrix_market(const char* path, bsp_host_csr* out);
/* write_matrix_market (:122-137): "coordinate real general", %.17g values. */
int bsp_write_matrix_market(const bsp_host_csr* A, const char* path);
/* load_permutation (:141-166; ReorderSpec::file, reorder.hpp:185-192): one
 * integer per line, perm[k] on line k; length and bijectivity checked. */
int bsp_load_permutation(const char* path, int64_t nrows, int32_t* perm_out);
int bsp_write_permutation(const int32_t* perm, int64_t n, const char* path);
void bsp_host_free_plain(void* p);

/* ------------------------------------------------------------------ */
/* seeded synthetic generators (BASELINE.json configs; DESIGN.md pins) */
/* ------------------------------------------------------------------ */
int bsp_gen_er(int64_t n, int32_t per_row, uint64_t seed, bsp_host_csr* out);
int bsp_gen_hidden_clusters(int64_t ntemplates, int32_t children, int32_t tcols,
                            double keep_p, double extra_mean, uint64_t seed,
                            uint64_t perm_seed, bsp_host_csr* out);
int bsp_gen_rmat(int32_t scale, int32_t edge_factor, double a, double b, double c,
                 uint64_t seed, bsp_host_csr* out);
int bsp_gen_stencil27(int32_t g, int64_t perm_seed /* <0: no permutation */, bsp_host_csr* out);

#ifdef __cplusplus
}
#endif
#endif /* BSP_H_ */
