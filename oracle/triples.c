/*
 * oracle/triples.c -- TEST INFRASTRUCTURE ONLY (NEXT-4).
 *
 * Plain CPU computation of the support of item triples, for the itemsets-of-size-3 extension
 * the paper leaves open.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library; it shares no code with paper_1102_1003_b200/.
 *
 * Definition implemented:
 *   supp({i,j,k}) = |S_i ∩ S_j ∩ S_k|     P:43-44 (support of an itemset = number of transactions
 *                                         containing it), vertical form P:56-58
 *   report triples i<j<k with supp >= s  P:43 (inclusive, reading #13)
 *
 * Two independent computations:
 *   oracle_triple_count / oracle_triples_list   three-finger sorted merge        (P:59 generalised)
 *   oracle_triples_horizontal                   for every transaction T_b and every triple
 *                                               a<c<d in T_b count +1            (P:62-63 generalised)
 *
 * Output: malloc'd uint32 quads (i, j, k, supp), i<j<k caller ids, sorted by (i, j, k).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* |a ∩ b ∩ c| for strictly increasing a, b, c: advance the smallest head. */
int64_t oracle_triple_count(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, const int32_t* c,
                            int64_t nc) {
    int64_t i = 0, j = 0, k = 0, n = 0;
    while (i < na && j < nb && k < nc) {
        int32_t x = a[i], y = b[j], z = c[k];
        if (x == y && y == z) {
            n++;
            i++;
            j++;
            k++;
        } else {
            int32_t mx = x > y ? x : y;
            if (z > mx) mx = z;
            if (x < mx) i++;
            if (y < mx) j++;
            if (z < mx) k++;
        }
    }
    return n;
}

/* Supports of an explicit list of triples (caller ids), one three-way merge each. */
void oracle_triples_list(const int64_t* offsets, const int32_t* tids, const int32_t* ti, const int32_t* tj,
                         const int32_t* tk, int64_t n_triples, uint32_t* out_supp) {
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t q = 0; q < n_triples; q++) {
        int32_t a = ti[q], b = tj[q], c = tk[q];
        out_supp[q] = (uint32_t)oracle_triple_count(tids + offsets[a], offsets[a + 1] - offsets[a],
                                                    tids + offsets[b], offsets[b + 1] - offsets[b],
                                                    tids + offsets[c], offsets[c + 1] - offsets[c]);
    }
}

typedef struct {
    uint32_t* v;
    int64_t n, cap;
} vec4;

static int vec4_push(vec4* b, uint32_t i, uint32_t j, uint32_t k, uint32_t s) {
    if (b->n + 1 > b->cap) {
        int64_t nc = b->cap ? 2 * b->cap : 64;
        uint32_t* nv = (uint32_t*)realloc(b->v, (size_t)nc * 4 * sizeof(uint32_t));
        if (!nv) return -1;
        b->v = nv;
        b->cap = nc;
    }
    uint32_t* o = b->v + 4 * b->n;
    o[0] = i;
    o[1] = j;
    o[2] = k;
    o[3] = s;
    b->n++;
    return 0;
}

static int cmp_i64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}

/*
 * Horizontal triple counting (P:62-63 generalised to 3-subsets).  Step 1: transpose the
 * selected items' tidlists into transactions T_b (selection indices, ascending).  Step 2: for
 * each first item u (rows across threads, thread-local counters, no atomics): for each b in
 * S_u, for each pair v < w in T_b with v > u: cnt[v][w] += 1.  Then emit supp >= threshold
 * (threshold >= 1) and reset.  The counters are a dense n_sel x n_sel array per thread, so
 * n_sel is limited to 4096 (returns -2 above).
 */
int64_t oracle_triples_horizontal(const int64_t* offsets, const int32_t* tids, int64_t m, const int32_t* items,
                                  int64_t n_sel, uint32_t threshold, uint32_t** out) {
    if (n_sel > 4096) return -2;
    if (threshold < 1) threshold = 1;
    int64_t* toff = (int64_t*)calloc((size_t)m + 1, sizeof(int64_t));
    if (!toff) return -1;
    for (int64_t u = 0; u < n_sel; u++) {
        int32_t a = items[u];
        for (int64_t k = offsets[a]; k < offsets[a + 1]; k++) toff[tids[k] + 1]++;
    }
    for (int64_t b = 0; b < m; b++) toff[b + 1] += toff[b];
    int64_t total = toff[m];
    int32_t* tu = (int32_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
    int64_t* fill = (int64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    if (!tu || !fill) {
        free(toff);
        free(tu);
        free(fill);
        return -1;
    }
    memcpy(fill, toff, (size_t)m * sizeof(int64_t));
    for (int64_t u = 0; u < n_sel; u++) {
        int32_t a = items[u];
        for (int64_t k = offsets[a]; k < offsets[a + 1]; k++) tu[fill[tids[k]]++] = (int32_t)u;
    }
    free(fill);
    vec4* rows = (vec4*)calloc((size_t)(n_sel > 0 ? n_sel : 1), sizeof(vec4));
    int failed = 0;
    #pragma omp parallel
    {
        const int64_t nn = n_sel > 0 ? n_sel * n_sel : 1;
        int32_t* cnt = (int32_t*)calloc((size_t)nn, sizeof(int32_t));
        int64_t cap = 1 << 16, nt = 0;
        int64_t* touched = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
        if (!cnt || !touched) failed = 1;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t u = 0; u < n_sel; u++) {
            if (!cnt || !touched || failed) continue;
            int32_t a = items[u];
            nt = 0;
            for (int64_t e = offsets[a]; e < offsets[a + 1]; e++) {
                int32_t b = tids[e];
                for (int64_t p = toff[b]; p < toff[b + 1]; p++) {
                    int32_t v = tu[p];
                    if (v <= u) continue;
                    for (int64_t q = p + 1; q < toff[b + 1]; q++) {
                        int32_t w = tu[q];  /* T_b ascending: w > v */
                        int64_t key = (int64_t)v * n_sel + w;
                        if (cnt[key]++ == 0) {
                            if (nt == cap) {
                                int64_t* nb = (int64_t*)realloc(touched, (size_t)(2 * cap) * sizeof(int64_t));
                                if (!nb) {
                                    failed = 1;
                                    break;
                                }
                                touched = nb;
                                cap *= 2;
                            }
                            touched[nt++] = key;
                        }
                    }
                }
            }
            qsort(touched, (size_t)nt, sizeof(int64_t), cmp_i64);
            for (int64_t q = 0; q < nt; q++) {
                int64_t key = touched[q];
                if ((uint32_t)cnt[key] >= threshold)
                    if (vec4_push(&rows[u], (uint32_t)a, (uint32_t)items[key / n_sel], (uint32_t)items[key % n_sel],
                                  (uint32_t)cnt[key]))
                        failed = 1;
                cnt[key] = 0;
            }
        }
        free(cnt);
        free(touched);
    }
    free(toff);
    free(tu);
    int64_t k = 0;
    for (int64_t r = 0; r < n_sel; r++) k += rows[r].n;
    uint32_t* o = failed ? NULL : (uint32_t*)malloc((size_t)(k > 0 ? k : 1) * 4 * sizeof(uint32_t));
    if (!o) {
        for (int64_t r = 0; r < n_sel; r++) free(rows[r].v);
        free(rows);
        return -1;
    }
    int64_t at = 0;
    for (int64_t r = 0; r < n_sel; r++) {
        if (rows[r].n) memcpy(o + 4 * at, rows[r].v, (size_t)rows[r].n * 4 * sizeof(uint32_t));
        at += rows[r].n;
        free(rows[r].v);
    }
    free(rows);
    *out = o;
    return k;
}
