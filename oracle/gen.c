/* gen.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the seeded R-MAT recipe of BASELINE.json cfg3/cfg5
 * (the product's generator is paper_2507_21253_b200/csrc/host_gen.cpp
 * gen_rmat; the recipe is pinned in DESIGN.md §5), so that bench.py's
 * reference arm (--impl reference) builds its input without loading the
 * product library.  tests/test_oracle.py checks that both generators give the
 * same matrix bit for bit.
 *
 * Recipe: m = n * edge_factor directed edges; edge e draws `scale` levels from
 * splitmix64(seed ^ e * 0xD1B54A32D192ED03) chained through splitmix64, each
 * level a quadrant by U[0,1) against (a, a+b, a+b+c); self-loops dropped; both
 * orientations kept (symmetrised); duplicates removed; the value of {i, j} is
 * U[0,1) from splitmix64(seed * golden ^ (min << 32 | max)).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static double unit_double(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

/* Returns 0, or -1 on bad sizes / allocation failure.  Outputs are malloc'd
 * (free with orc_free). */
int orc_gen_rmat(int32_t scale, int32_t edge_factor, double a, double b, double c, uint64_t seed,
                 int64_t* nrows_out, int64_t** rp_out, int32_t** ci_out, double** v_out) {
    if (scale < 1 || scale > 30 || edge_factor < 1) return -1;
    const int64_t n = (int64_t)1 << scale;
    const int64_t m = n * edge_factor;
    const double ab = a + b, abc = a + b + c;
    uint32_t* src = malloc((size_t)(2 * m) * sizeof(uint32_t));
    uint32_t* dst = malloc((size_t)(2 * m) * sizeof(uint32_t));
    int64_t* cnt = calloc((size_t)(n + 1), sizeof(int64_t));
    if (!src || !dst || !cnt) return -1;
    int64_t ne = 0;
    for (int64_t e = 0; e < m; ++e) {
        uint64_t s = splitmix64(seed ^ ((uint64_t)e * 0xD1B54A32D192ED03ull));
        uint64_t u = 0, v = 0;
        for (int32_t lvl = 0; lvl < scale; ++lvl) {
            s = splitmix64(s);
            const double r = unit_double(s);
            u <<= 1;
            v <<= 1;
            if (r < a) {
            } else if (r < ab) {
                v |= 1;
            } else if (r < abc) {
                u |= 1;
            } else {
                u |= 1;
                v |= 1;
            }
        }
        if (u == v) continue;
        src[ne] = (uint32_t)u;
        dst[ne++] = (uint32_t)v;
        src[ne] = (uint32_t)v;
        dst[ne++] = (uint32_t)u;
    }
    /* (row, col) order by two stable counting sorts: by column, then by row */
    uint32_t* s2 = malloc((size_t)ne * sizeof(uint32_t));
    uint32_t* d2 = malloc((size_t)ne * sizeof(uint32_t));
    int64_t* pos = malloc((size_t)(n + 1) * sizeof(int64_t));
    if (!s2 || !d2 || !pos) return -1;
    for (int pass = 0; pass < 2; ++pass) {
        const uint32_t* key = pass == 0 ? dst : s2;
        memset(pos, 0, (size_t)(n + 1) * sizeof(int64_t));
        for (int64_t i = 0; i < ne; ++i) ++pos[key[i] + 1];
        for (int64_t i = 0; i < n; ++i) pos[i + 1] += pos[i];
        if (pass == 0) {
            for (int64_t i = 0; i < ne; ++i) {
                const int64_t p = pos[dst[i]]++;
                s2[p] = src[i];
                d2[p] = dst[i];
            }
        } else {
            for (int64_t i = 0; i < ne; ++i) {
                const int64_t p = pos[s2[i]]++;
                src[p] = s2[i];
                dst[p] = d2[i];
            }
        }
    }
    free(s2);
    free(d2);
    free(pos);
    /* unique (row, col) pairs */
    int64_t nu = 0;
    for (int64_t i = 0; i < ne; ++i) {
        if (nu > 0 && src[nu - 1] == src[i] && dst[nu - 1] == dst[i]) continue;
        src[nu] = src[i];
        dst[nu] = dst[i];
        ++nu;
    }
    int64_t* rp = calloc((size_t)(n + 1), sizeof(int64_t));
    int32_t* ci = malloc((size_t)(nu > 0 ? nu : 1) * sizeof(int32_t));
    double* vv = malloc((size_t)(nu > 0 ? nu : 1) * sizeof(double));
    if (!rp || !ci || !vv) return -1;
    for (int64_t i = 0; i < nu; ++i) {
        ++rp[src[i] + 1];
        const uint64_t r = src[i], cc = dst[i];
        const uint64_t lo = r < cc ? r : cc, hi = r < cc ? cc : r;
        ci[i] = (int32_t)cc;
        vv[i] = unit_double(splitmix64((seed * 0x9E3779B97F4A7C15ull) ^ ((lo << 32) | hi)));
    }
    for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
    free(src);
    free(dst);
    free(cnt);
    *nrows_out = n;
    *rp_out = rp;
    *ci_out = ci;
    *v_out = vv;
    return 0;
}
