/* oracle.h — TEST INFRASTRUCTURE ONLY (see oracle.c). */
#ifndef ORACLE_H_
#define ORACLE_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t i, j;
    double score;
} orc_candidate;

typedef struct {
    uint64_t b_row_loads, a_inner_iters, placeholder_skips;
} orc_access_stats;

typedef struct {
    int64_t nclusters, nrows, ncols, ncolslots, nslots;
    int32_t* cluster_sizes;
    int64_t* cluster_col_ptr;
    int32_t* col_idx;
    int64_t* value_ptr;
    double* values;
    uint64_t* valid;
    int32_t* row_map;
} orc_cluster;

void orc_spgemm_symbolic(int64_t nrows, int64_t ncols_b, const int64_t* arp, const int32_t* acol,
                         const int64_t* brp, const int32_t* bcol, int64_t* counts);
int64_t orc_spgemm_rowwise(int64_t nrows, int64_t ncols_b, const int64_t* arp, const int32_t* acol,
                           const double* aval, const int64_t* brp, const int32_t* bcol,
                           const double* bval, int64_t* crp, int32_t** ccol_out,
                           double** cval_out);
double orc_jaccard(const int64_t* rp, const int32_t* col, int64_t i, int64_t j);
int64_t orc_spgemm_topk(int64_t nrows, const int64_t* arp, const int32_t* acol,
                        const int64_t* atrp, const int32_t* atcol, int32_t topk, double jacc_th,
                        orc_candidate** out);
void orc_build_csr_cluster(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* col,
                           const double* val, int64_t nclusters, const int64_t* cptr,
                           const int32_t* rows, orc_cluster* out);
int64_t orc_cluster_to_csr(const orc_cluster* m, int64_t* crp, int32_t** ccol_out,
                           double** cval_out);
void orc_spgemm_clusterwise(const orc_cluster* a, int64_t ncols_b, const int64_t* brp,
                            const int32_t* bcol, const double* bval, orc_cluster* c,
                            orc_access_stats* stats);
void orc_cluster_free(orc_cluster* c);
int64_t orc_merge_candidates(int64_t nrows, const int64_t* rp, const int32_t* col,
                             const orc_candidate* pairs, int64_t npairs, double jacc_th,
                             int32_t max_cluster, int32_t* cluster_of);
void orc_free(void* p);
/* gen.c: the seeded R-MAT recipe of cfg3/cfg5 (bench.py's reference arm input) */
int orc_gen_rmat(int32_t scale, int32_t edge_factor, double a, double b, double c, uint64_t seed,
                 int64_t* nrows_out, int64_t** rp_out, int32_t** ci_out, double** v_out);

#ifdef __cplusplus
}
#endif
#endif
