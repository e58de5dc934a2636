/*
 * oracle/pairs.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU computation of what the BatMap hot path
 * computes.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with
 * paper_1102_1003_b200/ (the CUDA path) and includes none of its headers.
 *
 * Definition implemented:
 *   supp({i,j}) = |S_i ∩ S_j|            P:43-44 ("support ... number of transactions
 *                                         that have S as a subset")
 *   report pairs i<j with supp >= s      P:43, north_star; threshold 0 = every pair
 *
 * Two independent computations:
 *   oracle_pairs_merge       sorted-list two-finger merge per pair
 *   oracle_pairs_horizontal  horizontal pair counting: for every transaction T_b and
 *                            every pair a<c in T_b count +1
 *
 * Output: malloc'd uint32 triples (i, j, supp), i<j in the caller's item ids, sorted
 * by (i, j).  Free with oracle_free().
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    uint32_t* v;
    int64_t n, cap;
} vec3;

static int vec3_push(vec3* b, uint32_t i, uint32_t j, uint32_t s) {
    if (b->n + 1 > b->cap) {
        int64_t nc = b->cap ? 2 * b->cap : 64;
        uint32_t* nv = (uint32_t*)realloc(b->v, (size_t)nc * 3 * sizeof(uint32_t));
        if (!nv) return -1;
        b->v = nv;
        b->cap = nc;
    }
    b->v[3 * b->n + 0] = i;
    b->v[3 * b->n + 1] = j;
    b->v[3 * b->n + 2] = s;
    b->n++;
    return 0;
}

/* Concatenate per-row buffers in row order into one malloc'd array. */
static int64_t concat_rows(vec3* rows, int64_t n_rows, uint32_t** out) {
    int64_t total = 0;
    for (int64_t r = 0; r < n_rows; r++) total += rows[r].n;
    uint32_t* o = (uint32_t*)malloc((size_t)(total > 0 ? total : 1) * 3 * sizeof(uint32_t));
    if (!o) return -1;
    int64_t k = 0;
    for (int64_t r = 0; r < n_rows; r++) {
        if (rows[r].n) memcpy(o + 3 * k, rows[r].v, (size_t)rows[r].n * 3 * sizeof(uint32_t));
        k += rows[r].n;
        free(rows[r].v);
    }
    *out = o;
    return total;
}

void oracle_free(void* p) { free(p); }

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* |a ∩ b| for strictly increasing a, b: the folklore two-finger merge. */
int64_t oracle_merge_count(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {
    int64_t i = 0, j = 0, c = 0;
    while (i < na && j < nb) {
        if (a[i] < b[j]) i++;
        else if (a[i] > b[j]) j++;
        else { c++; i++; j++; }
    }
    return c;
}

/* Supports of an explicit list of pairs (caller ids), one merge each. */
void oracle_merge_list(const int64_t* offsets, const int32_t* tids, const int32_t* pi,
                       const int32_t* pj, int64_t n_pairs, uint32_t* out_supp) {
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t k = 0; k < n_pairs; k++) {
        int32_t a = pi[k], c = pj[k];
        out_supp[k] = (uint32_t)oracle_merge_count(tids + offsets[a], offsets[a + 1] - offsets[a],
                                                   tids + offsets[c], offsets[c + 1] - offsets[c]);
    }
}

/*
 * Every pair (items[u], items[v]), row_begin <= u < row_end, u < v < n_sel, with
 * `items` strictly increasing caller ids.  Emits supp >= threshold (all if 0).
 */
int64_t oracle_pairs_merge(const int64_t* offsets, const int32_t* tids, const int32_t* items,
                           int64_t n_sel, int64_t row_begin, int64_t row_end, uint32_t threshold,
                           uint32_t** out) {
    if (row_end > n_sel) row_end = n_sel;
    if (row_begin < 0) row_begin = 0;
    int64_t n_rows = row_end > row_begin ? row_end - row_begin : 0;
    vec3* rows = (vec3*)calloc((size_t)(n_rows > 0 ? n_rows : 1), sizeof(vec3));
    if (!rows) return -1;
    int failed = 0;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < n_rows; r++) {
        int64_t u = row_begin + r;
        int32_t a = items[u];
        const int32_t* Sa = tids + offsets[a];
        int64_t na = offsets[a + 1] - offsets[a];
        for (int64_t v = u + 1; v < n_sel; v++) {
            int32_t c = items[v];
            int64_t s = oracle_merge_count(Sa, na, tids + offsets[c], offsets[c + 1] - offsets[c]);
            if ((uint64_t)s >= threshold)
                if (vec3_push(&rows[r], (uint32_t)a, (uint32_t)c, (uint32_t)s)) failed = 1;
        }
    }
    if (failed) {
        for (int64_t r = 0; r < n_rows; r++) free(rows[r].v);
        free(rows);
        return -1;
    }
    int64_t k = concat_rows(rows, n_rows, out);
    free(rows);
    return k;
}

static int cmp_i32(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

/*
 * Horizontal pair counting.  Step 1: transpose the selected items' tidlists
 * into transactions T_b (selection indices, ascending).  Step 2: for each first item
 * u (rows partitioned across threads, thread-local counters, no atomics): for each
 * b in S_u, for each v in T_b with v > u: cnt[v] += 1.  Then emit and reset.
 */
int64_t oracle_pairs_horizontal(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                                int64_t m, const int32_t* items, int64_t n_sel,
                                uint32_t threshold, uint32_t** out) {
    (void)n_items;
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
    if (!tu || !fill) { free(toff); free(tu); free(fill); return -1; }
    memcpy(fill, toff, (size_t)m * sizeof(int64_t));
    for (int64_t u = 0; u < n_sel; u++) {  /* u ascending => each T_b ascending */
        int32_t a = items[u];
        for (int64_t k = offsets[a]; k < offsets[a + 1]; k++) tu[fill[tids[k]]++] = (int32_t)u;
    }
    free(fill);

    vec3* rows = (vec3*)calloc((size_t)(n_sel > 0 ? n_sel : 1), sizeof(vec3));
    int failed = 0;
    #pragma omp parallel
    {
        int32_t* cnt = (int32_t*)calloc((size_t)(n_sel > 0 ? n_sel : 1), sizeof(int32_t));
        int32_t* touched = (int32_t*)malloc((size_t)(n_sel > 0 ? n_sel : 1) * sizeof(int32_t));
        if (!cnt || !touched) failed = 1;
        #pragma omp for schedule(dynamic, 4)
        for (int64_t u = 0; u < n_sel; u++) {
            if (!cnt || !touched) continue;
            int32_t a = items[u];
            int64_t nt = 0;
            for (int64_t k = offsets[a]; k < offsets[a + 1]; k++) {
                int32_t b = tids[k];
                for (int64_t q = toff[b]; q < toff[b + 1]; q++) {
                    int32_t v = tu[q];
                    if (v <= u) continue;
                    if (cnt[v]++ == 0) touched[nt++] = v;
                }
            }
            if (threshold == 0) {
                for (int64_t v = u + 1; v < n_sel; v++)
                    if (vec3_push(&rows[u], (uint32_t)a, (uint32_t)items[v], (uint32_t)cnt[v])) failed = 1;
            } else {
                qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
                for (int64_t q = 0; q < nt; q++) {
                    int32_t v = touched[q];
                    if ((uint32_t)cnt[v] >= threshold)
                        if (vec3_push(&rows[u], (uint32_t)a, (uint32_t)items[v], (uint32_t)cnt[v])) failed = 1;
                }
            }
            for (int64_t q = 0; q < nt; q++) cnt[touched[q]] = 0;
        }
        free(cnt);
        free(touched);
    }
    free(toff);
    free(tu);
    if (failed) {
        for (int64_t r = 0; r < n_sel; r++) free(rows[r].v);
        free(rows);
        return -1;
    }
    int64_t k = concat_rows(rows, n_sel, out);
    free(rows);
    return k;
}
