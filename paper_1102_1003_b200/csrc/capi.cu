// capi.cu -- the extern "C" boundary declared in include/batmap.h.
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "fimi.h"
#include "plan.h"

using namespace bm;

namespace {

void set_pool_threshold(int dev) {
    static bool done[64] = {false};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

void init_pool() {  // keep freed blocks in the stream-ordered pool (no re-mapping per call)
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) set_pool_threshold(dev);
}

void free_all(batmap_collection* h) {
    cudaStream_t st = h->stream;
    void* ptrs[] = {h->pos2orig_d, h->orig2pos_d, h->arena_d,   h->f_d,      h->fail_off_d, h->fail_tid_d,
                    h->fidx_of_tid_d, h->ab_off_d, h->ab_pos_d, h->cand_d,   h->ctr_d,      h->key_d,
                    h->val_d,     h->cub_tmp,    h->sel_arena_d, h->sel_idx_d, h->res_d,
                    h->cnt_d, h->tail_d, h->shard_fails_d};
    for (void* p : ptrs) dfree(p, st);
    if (h->k2prep) destroy_k2(h->k2prep, st);
    h->k2prep = nullptr;
}

bool full_selection(const batmap_collection* h, Selection* sel) {
    sel->classes = h->classes;
    sel->arena = h->arena_d;
    sel->f = h->f_d;
    sel->sel2pos = nullptr;
    sel->sel2orig = h->pos2orig_d;
    sel->n_sel = h->n;
    return true;
}

}  // namespace

extern "C" {

const char* batmap_last_error(void) { return get_error(); }

const char* batmap_version(void) { return "batmap-b200 0.1 (sm_100a)"; }

batmap_status batmap_build(const int64_t* offsets, const int32_t* tids, int64_t n_items, int64_t n_transactions,
                           const batmap_build_opts* opts, batmap_stream_t stream, batmap_handle* out) {
    return batmap_build_shard(offsets, tids, n_items, n_transactions, opts, 0, 1, stream, out);
}

// offsets_host: the same offsets already on the host (batmap_mine_host), or NULL: spares the
// build's read-back and lets its host planning overlap the tidlist upload.
static batmap_status build_impl(const int64_t* offsets, const int32_t* tids, int64_t n_items, int64_t n_transactions,
                                const batmap_build_opts* opts, int32_t part, int32_t n_parts, batmap_stream_t stream,
                                batmap_handle* out, const int64_t* offsets_host) {
    if (n_parts < 1 || part < 0 || part >= n_parts) {
        set_error("need 0 <= part < n_parts (got %d of %d)", part, n_parts);
        return BATMAP_E_INVALID;
    }
    if (!out) {
        set_error("out is NULL");
        return BATMAP_E_INVALID;
    }
    *out = nullptr;
    if (!offsets) {
        set_error("offsets is NULL");
        return BATMAP_E_INVALID;
    }
    if (n_items < 0 || n_transactions < 1) {
        set_error("need n_items >= 0 and n_transactions >= 1");
        return BATMAP_E_INVALID;
    }
    if (offsets_host) {
        if (!tids && n_items > 0 && offsets_host[n_items] != 0) {
            set_error("tids is NULL but offsets[n_items] = %lld", (long long)offsets_host[n_items]);
            return BATMAP_E_INVALID;
        }
    } else {
        BM_TRY(check_tids_device(offsets, tids, n_items, reinterpret_cast<cudaStream_t>(stream)));
    }
    if (n_items >= (1ll << 31) || n_transactions >= (1ll << 31)) {
        set_error("n_items and n_transactions must be < 2^31");
        return BATMAP_E_OVERFLOW;
    }
    uint32_t r_min = (opts && opts->r_min) ? opts->r_min : 128u;
    if (r_min < 4 || (r_min & (r_min - 1))) {
        set_error("r_min must be a power of two >= 4 (got %u)", r_min);
        return BATMAP_E_INVALID;
    }
    batmap_collection* h = new (std::nothrow) batmap_collection();
    if (!h) {
        set_error("host allocation failed");
        return BATMAP_E_NOMEM;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    h->stream = st;
    if (cudaGetDevice(&h->device) != cudaSuccess ||
        cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess) {
        cudaGetLastError();
        set_error("no CUDA device available");
        delete h;
        return BATMAP_E_CUDA;
    }
    set_pool_threshold(h->device);
    h->n = n_items;
    h->m = n_transactions;
    h->seed = opts ? opts->seed : 0;
    h->r_min = r_min;
    h->max_loop_opt = opts ? opts->max_loop : 0;
    batmap_status rc = build_collection(h, offsets, tids, opts, part, n_parts, st, offsets_host);
    if (rc != BATMAP_OK) {
        free_all(h);
        delete h;
        return rc;
    }
    *out = h;
    return BATMAP_OK;
}

batmap_status batmap_build_shard(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                                 int64_t n_transactions, const batmap_build_opts* opts, int32_t part,
                                 int32_t n_parts, batmap_stream_t stream, batmap_handle* out) {
    return build_impl(offsets, tids, n_items, n_transactions, opts, part, n_parts, stream, out, nullptr);
}

batmap_status batmap_shard_sizes(batmap_handle h, int32_t part, int64_t* words, int64_t* n_fail) {
    if (!h || !words || part < 0 || part >= h->shard_n_parts) {
        set_error("bad handle / part / words");
        return BATMAP_E_INVALID;
    }
    *words = shard_words(h, part, h->shard_n_parts);
    if (n_fail) *n_fail = part == h->shard_part ? h->shard_n_fail : -1;
    return BATMAP_OK;
}

batmap_status batmap_shard_export(batmap_handle h, uint32_t* words_out, int64_t words_capacity, uint64_t* fails_out,
                                  int64_t fails_capacity, batmap_stream_t stream) {
    if (!h || !h->shard_pending) {
        set_error("not a pending sharded build");
        return BATMAP_E_INVALID;
    }
    const int64_t need = shard_words(h, h->shard_part, h->shard_n_parts);
    if ((need && !words_out) || words_capacity < need || fails_capacity < h->shard_n_fail ||
        (h->shard_n_fail && !fails_out)) {
        set_error("export buffers too small: need %lld words and %lld failure records", (long long)need,
                  (long long)h->shard_n_fail);
        return BATMAP_E_CAPACITY;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    BM_TRY(shard_copy(h, h->shard_part, h->shard_n_parts, words_out, false, st));
    if (h->shard_n_fail)
        BM_CUDA(cudaMemcpyAsync(fails_out, h->shard_fails_d, h->shard_n_fail * sizeof(uint64_t),
                                cudaMemcpyDeviceToDevice, st));
    return BATMAP_OK;
}

batmap_status batmap_shard_import(batmap_handle h, const int64_t* offsets, const int32_t* tids,
                                  const uint32_t* words_all, int64_t stride_words, const uint64_t* fails_all,
                                  const int64_t* n_fails, int64_t stride_fails, batmap_stream_t stream) {
    if (!h || !h->shard_pending || !offsets || !n_fails) {
        set_error("not a pending sharded build, or NULL arguments");
        return BATMAP_E_INVALID;
    }
    const int N = h->shard_n_parts;
    for (int p = 0; p < N; ++p) {
        if (shard_words(h, p, N) > stride_words || n_fails[p] < 0 || n_fails[p] > stride_fails ||
            (p == h->shard_part && n_fails[p] != h->shard_n_fail)) {
            set_error("part %d: words/failure counts do not fit the strides or disagree with this part", p);
            return BATMAP_E_INVALID;
        }
        if ((p != h->shard_part && shard_words(h, p, N) && !words_all) || (n_fails[p] && !fails_all)) {
            set_error("NULL exchange buffer");
            return BATMAP_E_INVALID;
        }
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    BM_TRY(shard_import(h, offsets, tids, words_all, stride_words, fails_all, n_fails, stride_fails, st));
    BM_CUDA(cudaStreamSynchronize(st));
    return BATMAP_OK;
}

batmap_status batmap_pair_supports_ex(batmap_handle h, const int32_t* items, int64_t n_sel, uint32_t threshold,
                                      int32_t part, int32_t n_parts, uint32_t flags, batmap_triple* out,
                                      int64_t capacity, int64_t* n_out, batmap_stream_t stream) {
    if (h && h->shard_pending) {
        set_error("sharded build not complete: call batmap_shard_import first");
        return BATMAP_E_INVALID;
    }
    if (!h || !n_out || (!out && capacity > 0) || capacity < 0) {
        set_error("null handle / n_out / out");
        return BATMAP_E_INVALID;
    }
    if (n_parts < 1 || part < 0 || part >= n_parts) {
        set_error("need 0 <= part < n_parts");
        return BATMAP_E_INVALID;
    }
    if (items && n_sel < 0) {
        set_error("n_sel < 0");
        return BATMAP_E_INVALID;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    h->stream = st;
    const int64_t l0 = h->launches;
    const bool cached = h->res_n >= 0 && h->res_items == items && h->res_nsel == (items ? n_sel : -1) &&
                        h->res_thr == threshold && h->res_flags == flags && h->res_part == part &&
                        h->res_nparts == n_parts;
    if (!cached) {
        h->res_n = -1;
        rec(h, EV_P0, st);
        Selection sel;
        const bool frequent = (flags & BATMAP_PAIRS_FREQUENT) && threshold >= 1 && !(flags & BATMAP_PAIRS_RAW);
        if (frequent) {  // drop the items whose support |S_i| is below the threshold
            std::vector<int32_t> req;
            if (items) {
                req.resize(n_sel);
                if (n_sel) {
                    BM_CUDA(cudaMemcpyAsync(req.data(), items, n_sel * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                    BM_CUDA(cudaStreamSynchronize(st));
                }
            } else {
                req.resize(h->n);
                for (int64_t i = 0; i < h->n; ++i) req[i] = (int32_t)i;
            }
            std::vector<int32_t> keep;
            keep.reserve(req.size());
            for (int32_t i : req) {
                if (i < 0 || i >= h->n) {
                    set_error("items: id %d out of range [0, %lld)", i, (long long)h->n);
                    return BATMAP_E_INVALID;
                }
                if ((uint32_t)h->size_orig_h[i] >= threshold) keep.push_back(i);
            }
            if (!items && (int64_t)keep.size() == h->n) full_selection(h, &sel);
            else BM_TRY(gather_selection_host(h, keep, st, &sel));
        } else if (items) {
            BM_TRY(gather_selection(h, items, n_sel, st, &sel));
        } else {
            full_selection(h, &sel);
        }
        h->stats.n_selected = sel.n_sel;
        int64_t n_cand = 0, n_res = 0;
        h->stats.word_compares = h->stats.tile_compares = 0;
        h->stats.k2_kind = h->stats.k2_grid = 0;
        rec(h, EV_K20, st);  // re-recorded by run_intersect when a kernel runs
        rec(h, EV_K21, st);
        BM_TRY(run_intersect(h, sel, threshold, part, n_parts, flags, st, &n_cand));
        rec(h, EV_K30, st);
        BM_TRY(run_finalize(h, sel, n_cand, threshold, flags, st, &n_res));
        rec(h, EV_P1, st);
        h->pairs_timed = true;
        h->stats.n_candidates = n_cand;
        h->stats.n_results = n_res;
        h->res_n = n_res;
        h->res_items = items;
        h->res_nsel = items ? n_sel : -1;
        h->res_thr = threshold;
        h->res_flags = flags;
        h->res_part = part;
        h->res_nparts = n_parts;
    }
    *n_out = h->res_n;
    if (h->res_n > capacity) {
        set_error("capacity %lld < %lld results", (long long)capacity, (long long)h->res_n);
        return BATMAP_E_CAPACITY;
    }
    if (h->res_n > 0)
        BM_CUDA(cudaMemcpyAsync(out, h->res_d, h->res_n * sizeof(batmap_triple), cudaMemcpyDeviceToDevice, st));
    h->res_n = -1;  // consumed; the next call recomputes
    h->stats.launches_pairs = h->launches - l0;
    return BATMAP_OK;
}

batmap_status batmap_pair_supports(batmap_handle h, const int32_t* items, int64_t n_sel, uint32_t threshold,
                                   batmap_triple* out, int64_t capacity, int64_t* n_out, batmap_stream_t stream) {
    return batmap_pair_supports_ex(h, items, n_sel, threshold, 0, 1, 0u, out, capacity, n_out, stream);
}

batmap_status batmap_pair_supports_part(batmap_handle h, const int32_t* items, int64_t n_sel, uint32_t threshold,
                                        int32_t part, int32_t n_parts, batmap_triple* out, int64_t capacity,
                                        int64_t* n_out, batmap_stream_t stream) {
    return batmap_pair_supports_ex(h, items, n_sel, threshold, part, n_parts, 0u, out, capacity, n_out, stream);
}

batmap_status batmap_info(batmap_handle h, batmap_info_t* info) {
    if (!h || !info) {
        set_error("null handle / info");
        return BATMAP_E_INVALID;
    }
    info->s_shift = h->s;
    info->n_classes = (int32_t)h->classes.size();
    info->U = h->U;
    info->r0 = h->r0;
    info->n_items = h->n;
    info->n_transactions = h->m;
    info->arena_bytes = h->arena_bytes_raw;
    info->n_failures = h->n_fail;
    info->n_failed_tids = h->n_ftid;
    return BATMAP_OK;
}

void batmap_destroy(batmap_handle h) {
    if (!h) return;
    free_all(h);
    if (h->ev_ok)
        for (int i = 0; i < EV_COUNT; ++i) cudaEventDestroy(h->ev[i]);
    delete h;
}

static double ev_ms(batmap_collection* h, int a, int b) {
    float ms = 0.f;
    if (cudaEventSynchronize(h->ev[b]) != cudaSuccess || cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]) != cudaSuccess) {
        cudaGetLastError();
        return -1.0;
    }
    return (double)ms;
}

batmap_status batmap_stats(batmap_handle h, batmap_stats_t* out) {
    if (!h || !out) {
        set_error("null handle / out");
        return BATMAP_E_INVALID;
    }
    if (h->ev_ok && h->build_timed) {
        h->stats.build_ms = ev_ms(h, EV_B0, EV_B1);
        h->stats.k1_insert_ms = ev_ms(h, EV_I0, EV_I1);
        h->stats.k1_encode_ms = ev_ms(h, EV_E0, EV_E1);
        h->stats.build_pre_ms = ev_ms(h, EV_B0, EV_I0);
        h->stats.build_post_ms = ev_ms(h, EV_E1, EV_B1);
    }
    if (h->ev_ok && h->pairs_timed) {
        h->stats.pairs_ms = ev_ms(h, EV_P0, EV_P1);
        h->stats.k2_ms = ev_ms(h, EV_K20, EV_K21);
        h->stats.k3_ms = ev_ms(h, EV_K30, EV_P1);
    }
    *out = h->stats;
    return BATMAP_OK;
}

batmap_status batmap_dense_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                                         int64_t n_transactions, const int32_t* items, int64_t n_sel,
                                         uint32_t threshold, batmap_triple* out, int64_t capacity, int64_t* n_out,
                                         double* gemm_ms, batmap_stream_t stream) {
    if (!offsets || !n_out || (!out && capacity > 0) || n_items < 0 ||
        n_transactions < 1 || (items && n_sel < 0)) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    if (n_items >= (1ll << 31) || n_transactions >= (1ll << 31)) {
        set_error("n_items and n_transactions must be < 2^31");
        return BATMAP_E_OVERFLOW;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    init_pool();
    BM_TRY(check_tids_device(offsets, tids, n_items, st));
    if (items && n_sel) {  // validate the selection on the host
        std::vector<int32_t> it(n_sel);
        BM_CUDA(cudaMemcpyAsync(it.data(), items, n_sel * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        std::sort(it.begin(), it.end());
        for (int64_t k = 0; k < n_sel; ++k)
            if (it[k] < 0 || it[k] >= n_items || (k && it[k] == it[k - 1])) {
                set_error("items must be distinct ids in [0, n_items)");
                return BATMAP_E_INVALID;
            }
    }
    return dense_pair_supports(offsets, tids, n_items, n_transactions, items, n_sel, threshold, out, capacity, n_out,
                               gemm_ms, st);
}

batmap_status batmap_merge_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                                         int64_t n_transactions, const int32_t* items, int64_t n_sel,
                                         uint32_t threshold, batmap_triple* out, int64_t capacity, int64_t* n_out,
                                         double* kernel_ms, int64_t* merge_steps, batmap_stream_t stream) {
    if (!offsets || !n_out || (!out && capacity > 0) || n_items < 0 ||
        n_transactions < 1 || (items && n_sel < 0)) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    if (n_items >= (1ll << 31) || n_transactions >= (1ll << 31)) {
        set_error("n_items and n_transactions must be < 2^31");
        return BATMAP_E_OVERFLOW;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    init_pool();
    BM_TRY(check_tids_device(offsets, tids, n_items, st));
    if (items && n_sel) {  // validate the selection on the host
        std::vector<int32_t> it(n_sel);
        BM_CUDA(cudaMemcpyAsync(it.data(), items, n_sel * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        std::sort(it.begin(), it.end());
        for (int64_t k = 0; k < n_sel; ++k)
            if (it[k] < 0 || it[k] >= n_items || (k && it[k] == it[k - 1])) {
                set_error("items must be distinct ids in [0, n_items)");
                return BATMAP_E_INVALID;
            }
    }
    return merge_pair_supports(offsets, tids, n_items, items, n_sel, threshold, out, capacity, n_out, kernel_ms,
                               merge_steps, st);
}

batmap_status batmap_sort_triples(batmap_triple* triples, int64_t n, batmap_stream_t stream) {
    if (!triples && n > 0) {
        set_error("null triples");
        return BATMAP_E_INVALID;
    }
    return sort_triples(triples, n, reinterpret_cast<cudaStream_t>(stream));
}

batmap_status batmap_mine_host(const int64_t* offsets, const int32_t* tids, int64_t n_items, int64_t n_transactions,
                               const batmap_build_opts* opts, const int32_t* items, int64_t n_sel,
                               uint32_t threshold, batmap_triple* out, int64_t capacity, int64_t* n_out,
                               batmap_stream_t stream) {
    if (!offsets || !n_out || (!out && capacity > 0) || n_items < 0) {
        set_error("null argument");
        return BATMAP_E_INVALID;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nnz = offsets[n_items];
    int64_t* off_d = nullptr;
    int32_t *tids_d = nullptr, *items_d = nullptr;
    batmap_triple* out_d = nullptr;
    batmap_handle h = nullptr;
    batmap_status rc = BATMAP_OK;
    auto cleanup = [&]() {
        batmap_destroy(h);
        dfree(off_d, st);
        dfree(tids_d, st);
        dfree(items_d, st);
        dfree(out_d, st);
    };
    if ((rc = dalloc_t(&off_d, n_items + 1, st)) != BATMAP_OK || (rc = dalloc_t(&tids_d, nnz, st)) != BATMAP_OK ||
        (items && (rc = dalloc_t(&items_d, n_sel, st)) != BATMAP_OK) ||
        (rc = dalloc_t(&out_d, std::max<int64_t>(capacity, 1), st)) != BATMAP_OK) {
        cleanup();
        return rc;
    }
    if (cudaMemcpyAsync(off_d, offsets, (n_items + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        (nnz && cudaMemcpyAsync(tids_d, tids, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, st) != cudaSuccess) ||
        (items && n_sel &&
         cudaMemcpyAsync(items_d, items, n_sel * sizeof(int32_t), cudaMemcpyHostToDevice, st) != cudaSuccess)) {
        set_error("H2D copy failed: %s", cudaGetErrorString(cudaGetLastError()));
        cleanup();
        return BATMAP_E_CUDA;
    }
    rc = build_impl(off_d, tids_d, n_items, n_transactions, opts, 0, 1, stream, &h, offsets);
    if (rc == BATMAP_OK)
        rc = batmap_pair_supports(h, items ? items_d : nullptr, n_sel, threshold, out_d, capacity, n_out, stream);
    if (rc == BATMAP_OK && *n_out > 0) {
        if (cudaMemcpyAsync(out, out_d, *n_out * sizeof(batmap_triple), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            set_error("D2H copy failed: %s", cudaGetErrorString(cudaGetLastError()));
            rc = BATMAP_E_CUDA;
        }
    }
    cleanup();
    return rc;
}

batmap_status batmap_export_entries(batmap_handle h, int32_t item, uint8_t* out, int64_t capacity, int64_t* r_out) {
    if (!h || !out || !r_out || item < 0 || item >= h->n) {
        set_error("bad handle / item / out");
        return BATMAP_E_INVALID;
    }
    const int64_t pos = h->orig2pos_h[item];
    const ClassInfo* c = nullptr;
    for (const ClassInfo& ci : h->classes)
        if (pos >= ci.first && pos < ci.first + ci.n) c = &ci;
    *r_out = c->r;
    if (capacity < 3ll * c->r) {
        set_error("capacity %lld < 3 r = %lld", (long long)capacity, 3ll * c->r);
        return BATMAP_E_CAPACITY;
    }
    const uint32_t* src = h->arena_d + c->word_off + (pos - c->first);
    BM_CUDA(cudaMemcpy2DAsync(out, 4, src, (size_t)c->n_pad * 4, 4, (size_t)c->W, cudaMemcpyDeviceToHost, h->stream));
    BM_CUDA(cudaStreamSynchronize(h->stream));
    return BATMAP_OK;
}

batmap_status batmap_export_failures(batmap_handle h, int32_t* items, int32_t* tids, int64_t capacity,
                                     int64_t* n_out) {
    if (!h || !n_out || ((!items || !tids) && capacity > 0)) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    *n_out = h->n_fail;
    if (capacity < h->n_fail) {
        set_error("capacity %lld < %lld failures", (long long)capacity, (long long)h->n_fail);
        return BATMAP_E_CAPACITY;
    }
    if (h->n_fail == 0) return BATMAP_OK;
    std::vector<int64_t> off(h->n + 1);
    std::vector<int32_t> ft(h->n_fail);
    BM_CUDA(cudaMemcpyAsync(off.data(), h->fail_off_d, (h->n + 1) * 8, cudaMemcpyDeviceToHost, h->stream));
    BM_CUDA(cudaMemcpyAsync(ft.data(), h->fail_tid_d, h->n_fail * 4, cudaMemcpyDeviceToHost, h->stream));
    BM_CUDA(cudaStreamSynchronize(h->stream));
    std::vector<std::pair<int32_t, int32_t>> rec;
    rec.reserve(h->n_fail);
    for (int64_t p = 0; p < h->n; ++p)
        for (int64_t q = off[p]; q < off[p + 1]; ++q) rec.emplace_back(h->pos2orig_h[p], ft[q]);
    std::sort(rec.begin(), rec.end());
    for (size_t k = 0; k < rec.size(); ++k) {
        items[k] = rec[k].first;
        tids[k] = rec[k].second;
    }
    return BATMAP_OK;
}

batmap_status batmap_swar_device(const uint32_t* x, const uint32_t* y, int64_t n, uint32_t* out,
                                 batmap_stream_t stream) {
    if ((!x || !y || !out) && n > 0) {
        set_error("null argument");
        return BATMAP_E_INVALID;
    }
    return swar_device(x, y, n, out, reinterpret_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------------ NEXT-3: FIMI ingestion
batmap_status batmap_fimi_parse(const uint8_t* text, int64_t n_bytes, batmap_stream_t stream, batmap_fimi_handle* out,
                                int64_t* bad_line) {
    if (!out || !bad_line || n_bytes < 0 || (!text && n_bytes > 0)) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    *out = nullptr;
    *bad_line = -1;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    init_pool();
    batmap_fimi* h = new (std::nothrow) batmap_fimi();
    if (!h) {
        set_error("host allocation");
        return BATMAP_E_NOMEM;
    }
    const batmap_status rc = fimi_parse(text, n_bytes, st, h, bad_line);
    if (rc != BATMAP_OK) {
        batmap_fimi_destroy(h);
        return rc;
    }
    *out = h;
    return BATMAP_OK;
}

batmap_status batmap_fimi_info(batmap_fimi_handle h, int64_t* n_items, int64_t* nnz, int64_t* n_transactions) {
    if (!h || !n_items || !nnz || !n_transactions) {
        set_error("null argument");
        return BATMAP_E_INVALID;
    }
    *n_items = h->n_items;
    *nnz = h->nnz;
    *n_transactions = h->m;
    return BATMAP_OK;
}

batmap_status batmap_fimi_filter(batmap_fimi_handle h, uint32_t min_support, batmap_stream_t stream) {
    if (!h) {
        set_error("null handle");
        return BATMAP_E_INVALID;
    }
    return fimi_filter(h, min_support, reinterpret_cast<cudaStream_t>(stream));
}

batmap_status batmap_fimi_export(batmap_fimi_handle h, int64_t* offsets, int32_t* tids, uint32_t* labels,
                                 batmap_stream_t stream) {
    if (!h) {
        set_error("null handle");
        return BATMAP_E_INVALID;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (offsets)
        BM_CUDA(cudaMemcpyAsync(offsets, h->off_d, (h->n_items + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    if (tids && h->nnz) BM_CUDA(cudaMemcpyAsync(tids, h->tids_d, h->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    if (labels && h->n_items)
        BM_CUDA(cudaMemcpyAsync(labels, h->labels_d, h->n_items * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    return BATMAP_OK;
}

void batmap_fimi_destroy(batmap_fimi_handle h) {
    if (!h) return;
    dfree(h->off_d, nullptr);
    dfree(h->tids_d, nullptr);
    dfree(h->labels_d, nullptr);
    delete h;
}

batmap_status batmap_frequent_items(const int64_t* offsets, int64_t n_items, uint32_t min_support, int32_t* items_out,
                                    int64_t* n_out, batmap_stream_t stream) {
    if (!n_out || n_items < 0 || (n_items > 0 && (!offsets || !items_out))) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    if (n_items >= (1ll << 31)) {
        set_error("n_items must be < 2^31");
        return BATMAP_E_OVERFLOW;
    }
    init_pool();
    return frequent_items(offsets, n_items, min_support, items_out, n_out, reinterpret_cast<cudaStream_t>(stream));
}

batmap_status batmap_select_csr(const int64_t* offsets, const int32_t* tids, int64_t n_items, const int32_t* items,
                                int64_t n_sel, int64_t* offsets_out, int32_t* tids_out, int64_t tids_capacity,
                                int64_t* nnz_out, batmap_stream_t stream) {
    if (!nnz_out || !offsets_out || n_items < 0 || n_sel < 0 || (n_sel && (!offsets || !tids || !items)) ||
        tids_capacity < 0 || (tids_capacity && !tids_out)) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    init_pool();
    return select_csr(offsets, tids, items, n_sel, offsets_out, tids_out, tids_capacity, nnz_out,
                      reinterpret_cast<cudaStream_t>(stream));
}

static bool promote_enabled() {
    const char* e = getenv("BATMAP_K2_PROMOTE");
    return !(e && e[0] == '0');
}

static batmap_status plan_classes(int32_t n_classes, const int64_t* class_n, const int64_t* class_w,
                                  std::vector<ClassInfo>* out) {
    std::vector<ClassInfo>& cls = *out;
    cls.assign(n_classes, ClassInfo{});
    int64_t first = 0;
    for (int a = 0; a < n_classes; ++a) {
        if (class_w[a] <= 0 || class_w[a] % kChunk || (a && class_w[a] < class_w[a - 1]) || class_n[a] < 0) {
            set_error("class_w must be ascending multiples of %d", kChunk);
            return BATMAP_E_INVALID;
        }
        cls[a].first = first;
        cls[a].n = (int32_t)class_n[a];
        cls[a].W = (int32_t)class_w[a];
        cls[a].n_pad = (int32_t)((class_n[a] + kPadItems - 1) / kPadItems * kPadItems);
        first += class_n[a];
    }
    return BATMAP_OK;
}

batmap_status batmap_plan_groups(int32_t n_classes, const int64_t* class_n, const int64_t* class_w,
                                 int32_t* group_of) {
    if (n_classes < 0 || (n_classes && (!class_n || !class_w || !group_of))) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    std::vector<ClassInfo> cls;
    BM_TRY(plan_classes(n_classes, class_n, class_w, &cls));
    Plan pl;
    const int tn = choose_tn(cls, true, promote_enabled());
    plan_work(cls, 0, 1, (tn == 64 ? 4 : 2) * 148, true, true, promote_enabled(), &pl, tn);
    for (int a = 0; a < n_classes; ++a) group_of[a] = pl.eff_of[a];
    return BATMAP_OK;
}

batmap_status batmap_plan_tile(int32_t n_classes, const int64_t* class_n, const int64_t* class_w, int32_t* tile_rows,
                               int32_t* tile_cols) {
    if (n_classes < 0 || (n_classes && (!class_n || !class_w)) || !tile_rows || !tile_cols) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    std::vector<ClassInfo> cls;
    BM_TRY(plan_classes(n_classes, class_n, class_w, &cls));
    *tile_rows = kTile;
    *tile_cols = choose_tn(cls, true, promote_enabled());
    return BATMAP_OK;
}

batmap_status batmap_plan_work(int32_t n_classes, const int64_t* class_n, const int64_t* class_w, int32_t part,
                               int32_t n_parts, int32_t grid_cap, int32_t* items, int64_t capacity, int64_t* n_items,
                               int64_t* word_compares, int64_t* tile_compares) {
    if (n_classes < 0 || (n_classes && (!class_n || !class_w)) || !n_items || !word_compares || !tile_compares ||
        n_parts < 1 || part < 0 || part >= n_parts || grid_cap < 0) {
        set_error("bad arguments");
        return BATMAP_E_INVALID;
    }
    std::vector<ClassInfo> cls;
    BM_TRY(plan_classes(n_classes, class_n, class_w, &cls));
    Plan pl;
    const int tn = choose_tn(cls, true, promote_enabled());
    plan_work(cls, part, n_parts, grid_cap ? grid_cap : (tn == 64 ? 4 : 2) * 148, true, true, promote_enabled(), &pl,
              tn);
    *n_items = (int64_t)pl.work.size();
    *word_compares = pl.word_compares;
    *tile_compares = pl.tile_compares;
    if (capacity < *n_items) {
        set_error("capacity %lld < %lld work items", (long long)capacity, (long long)*n_items);
        return BATMAP_E_CAPACITY;
    }
    for (size_t k = 0; k < pl.work.size(); ++k) {
        const Work& w = pl.work[k];
        const Rect& r = pl.rects[w.rect];
        int32_t* o = items + 8 * k;
        o[0] = r.cls_a;
        o[1] = r.cls_b;
        o[2] = w.ti;
        o[3] = w.tj;
        o[4] = w.k0;
        o[5] = w.k1;
        o[6] = r.R;
        o[7] = r.acc;
    }
    return BATMAP_OK;
}

}  // extern "C"
