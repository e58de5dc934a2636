// finalize.cu -- ★K3: exact failed-insertion corrections, re-threshold, id mapping, sort
// (P:469-474), plus the gather of an item subset into a compact selection.
//
// A candidate (i, j, c) from the intersection kernel satisfies c + f_i + f_j >= s.  Its
// exact support is c + |{b in S_i ∩ S_j : (i,b) in F or (j,b) in F}| (P:471-473 with set
// semantics, reading #11):
//   corr = #{b in Fail(i) : j in A_b} + #{b in Fail(j) : i in A_b and b not in Fail(i)},
// A_b being the (sorted) items of a failed transaction b.  Pairs with
// c + corr >= s are mapped to caller ids (i < j) and radix-sorted by (i, j).
#include <algorithm>
#include <cub/cub.cuh>

#include "common.cuh"

namespace bm {

__device__ __forceinline__ bool bsearch_i32(const int32_t* __restrict__ a, int64_t lo, int64_t hi, int32_t v) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        int32_t x = a[mid];
        if (x == v) return true;
        if (x < v) lo = mid + 1;
        else hi = mid;
    }
    return false;
}

struct FailView {
    const int32_t* f;         // per position
    const int64_t* fail_off;  // n+1
    const int32_t* fail_tid;  // sorted per position
    const int32_t* fidx;      // per tid, -1 if not failed
    const int64_t* ab_off;
    const int32_t* ab_pos;    // sorted per failed tid
};

__global__ void __launch_bounds__(256) k3_correct(const Cand* __restrict__ cand, int64_t n,
                                                  const int32_t* __restrict__ sel2pos,
                                                  const int32_t* __restrict__ sel2orig, FailView fv,
                                                  uint32_t thr, uint32_t raw, uint64_t n_ids, uint64_t* __restrict__ keys,
                                                  uint32_t* __restrict__ vals,
                                                  unsigned long long* __restrict__ ctr) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const Cand cd = cand[k];
    const int32_t pi = sel2pos ? sel2pos[cd.i] : (int32_t)cd.i;
    const int32_t pj = sel2pos ? sel2pos[cd.j] : (int32_t)cd.j;
    uint64_t supp = cd.c;
    if (!raw && (fv.f[pi] | fv.f[pj])) {
        const int64_t ib = fv.fail_off[pi], ie = fv.fail_off[pi + 1];
        const int64_t jb = fv.fail_off[pj], je = fv.fail_off[pj + 1];
        uint32_t corr = 0;
        for (int64_t q = ib; q < ie; ++q) {  // b in Fail(i), j in A_b
            const int32_t fk = fv.fidx[fv.fail_tid[q]];
            corr += bsearch_i32(fv.ab_pos, fv.ab_off[fk], fv.ab_off[fk + 1], pj);
        }
        for (int64_t q = jb; q < je; ++q) {  // b in Fail(j), i in A_b, b not already counted
            const int32_t b = fv.fail_tid[q];
            const int32_t fk = fv.fidx[b];
            if (bsearch_i32(fv.ab_pos, fv.ab_off[fk], fv.ab_off[fk + 1], pi) &&
                !bsearch_i32(fv.fail_tid, ib, ie, b))
                ++corr;
        }
        supp += corr;
    }
    if (supp < thr) return;
    uint32_t oi = (uint32_t)sel2orig[cd.i], oj = (uint32_t)sel2orig[cd.j];
    if (oi > oj) {
        uint32_t t = oi;
        oi = oj;
        oj = t;
    }
    const unsigned long long at = atomicAdd(ctr, 1ull);
    keys[at] = (uint64_t)oi * n_ids + oj;  // < n_ids^2: fewer radix passes than (i << 32 | j)
    vals[at] = (uint32_t)supp;
}

// keys are i * n_ids + j, or (i << 32 | j) when n_ids == 0 (batmap_sort_triples)
__global__ void k3_emit(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                        uint64_t n_ids, batmap_triple* __restrict__ out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint64_t key = keys[k];
    batmap_triple t;
    if (n_ids) {
        t.i = (uint32_t)(key / n_ids);
        t.j = (uint32_t)(key - (uint64_t)t.i * n_ids);
    } else {
        t.i = (uint32_t)(key >> 32);
        t.j = (uint32_t)key;
    }
    t.support = vals[k];
    out[k] = t;
}

static int bits_for(uint64_t v) {
    int l = 1;
    while ((1ull << l) <= v) ++l;
    return l;
}

batmap_status run_finalize(batmap_collection* h, const Selection& sel, int64_t n_cand, uint32_t threshold,
                           uint32_t flags, cudaStream_t st, int64_t* n_res) {
    *n_res = 0;
    if (n_cand == 0) return BATMAP_OK;
    // keys/vals double buffers
    if (h->kv_cap < n_cand) {
        dfree(h->key_d, st);
        dfree(h->val_d, st);
        h->key_d = nullptr;
        h->val_d = nullptr;
        int64_t c = n_cand + n_cand / 4 + 1024;
        BM_TRY(dalloc_t(&h->key_d, 2 * c, st));
        BM_TRY(dalloc_t(&h->val_d, 2 * c, st));
        h->kv_cap = c;
    }
    uint64_t* k0 = h->key_d;
    uint64_t* k1 = h->key_d + h->kv_cap;
    uint32_t* v0 = h->val_d;
    uint32_t* v1 = h->val_d + h->kv_cap;
    FailView fv{h->f_d, h->fail_off_d, h->fail_tid_d, h->fidx_of_tid_d, h->ab_off_d, h->ab_pos_d};
    BM_CUDA(cudaMemsetAsync(h->ctr_d + 1, 0, sizeof(unsigned long long), st));
    h->launches += 1;
    k3_correct<<<(unsigned)((n_cand + 255) / 256), 256, 0, st>>>(
        h->cand_d, n_cand, sel.sel2pos, sel.sel2orig, fv, threshold, (flags & BATMAP_PAIRS_RAW) ? 1u : 0u,
        (uint64_t)h->n, k0, v0, h->ctr_d + 1);
    BM_CUDA(cudaGetLastError());
    unsigned long long cnt = 0;
    BM_TRY(read_scalar(st, h->ctr_d + 1, &cnt));
    const int64_t K = (int64_t)cnt;
    *n_res = K;
    BM_TRY(ensure(&h->res_d, &h->res_cap, std::max<int64_t>(K, 1), st));
    if (K == 0) return BATMAP_OK;
    const int kb = bits_for((uint64_t)h->n * (uint64_t)h->n);  // keys i * n + j < n^2
    cub::DoubleBuffer<uint64_t> dk(k0, k1);
    cub::DoubleBuffer<uint32_t> dv(v0, v1);
    size_t tb = 0;
    BM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)K, 0, kb, st));
    if (!h->cub_tmp || h->cub_tmp_bytes < tb) {
        dfree(h->cub_tmp, st);
        h->cub_tmp = nullptr;
        BM_TRY(dalloc(&h->cub_tmp, tb + tb / 4 + 4096, st));
        h->cub_tmp_bytes = tb + tb / 4 + 4096;
    }
    BM_CUDA(cub::DeviceRadixSort::SortPairs(h->cub_tmp, tb, dk, dv, (int)K, 0, kb, st));
    h->launches += 2;
    k3_emit<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(dk.Current(), dv.Current(), K, (uint64_t)h->n, h->res_d);
    BM_CUDA(cudaGetLastError());
    return BATMAP_OK;
}

__global__ void k_triple_keys(const batmap_triple* __restrict__ t, int64_t n, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    keys[k] = ((uint64_t)t[k].i << 32) | t[k].j;
    vals[k] = t[k].support;
}

batmap_status sort_triples(batmap_triple* t, int64_t n, cudaStream_t st) {
    if (n <= 1) return BATMAP_OK;
    uint64_t* kb = nullptr;
    uint32_t* vb = nullptr;
    void* tmp = nullptr;
    Scratch scratch(st);
    scratch.own(&kb);
    scratch.own(&vb);
    scratch.own(&tmp);
    BM_TRY(dalloc_t(&kb, 2 * n, st));
    BM_TRY(dalloc_t(&vb, 2 * n, st));
    k_triple_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(t, n, kb, vb);
    cub::DoubleBuffer<uint64_t> dk(kb, kb + n);
    cub::DoubleBuffer<uint32_t> dv(vb, vb + n);
    size_t tb = 0;
    BM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n, 0, 64, st));
    BM_TRY(dalloc(&tmp, tb + 16, st));
    BM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)n, 0, 64, st));
    k3_emit<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dk.Current(), dv.Current(), n, 0, t);
    BM_CUDA(cudaGetLastError());
    return BATMAP_OK;
}

// ------------------------------------------------------------------ selection of an item subset
__global__ void k_gather_cols(const uint32_t* __restrict__ arena, int64_t src_word_off, int32_t src_npad,
                              int64_t src_first, const int32_t* __restrict__ sel2pos, int64_t sel_first,
                              int32_t n, int32_t n_pad, int32_t W, uint32_t* __restrict__ dst) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)W * n_pad) return;
    const int w = (int)(idx / n_pad);
    const int c = (int)(idx - (int64_t)w * n_pad);
    uint32_t v = kNullWord;
    if (c < n) {
        const int64_t col = sel2pos[sel_first + c] - src_first;
        v = arena[src_word_off + (int64_t)w * src_npad + col];
    }
    dst[idx] = v;
}

__global__ void k_gather_meta(const int32_t* __restrict__ sel2pos, int64_t n, const int32_t* __restrict__ pos2orig,
                              const int32_t* __restrict__ f, int32_t* __restrict__ sel2orig,
                              int32_t* __restrict__ fsel) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t p = sel2pos[k];
    sel2orig[k] = pos2orig[p];
    fsel[k] = f[p];
}

batmap_status gather_selection(batmap_collection* h, const int32_t* items_d, int64_t n_sel, cudaStream_t st,
                               Selection* sel) {
    std::vector<int32_t> items(n_sel);
    if (n_sel) {
        BM_CUDA(cudaMemcpyAsync(items.data(), items_d, n_sel * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
    }
    return gather_selection_host(h, items, st, sel);
}

batmap_status gather_selection_host(batmap_collection* h, const std::vector<int32_t>& items, cudaStream_t st,
                                    Selection* sel) {
    const int64_t n_sel = (int64_t)items.size();
    std::vector<int32_t> pos(n_sel);
    for (int64_t k = 0; k < n_sel; ++k) {
        if (items[k] < 0 || items[k] >= h->n) {
            set_error("items[%lld] = %d out of range [0, %lld)", (long long)k, items[k], (long long)h->n);
            return BATMAP_E_INVALID;
        }
        pos[k] = h->orig2pos_h[items[k]];
    }
    std::sort(pos.begin(), pos.end());
    for (int64_t k = 1; k < n_sel; ++k)
        if (pos[k] == pos[k - 1]) {
            set_error("items contains duplicate id %d", h->pos2orig_h[pos[k]]);
            return BATMAP_E_INVALID;
        }
    sel->classes.clear();
    sel->n_sel = n_sel;
    int64_t word_off = 0;
    std::vector<int> src_class;
    size_t ci = 0;
    for (int64_t k = 0; k < n_sel;) {
        while (h->classes[ci].first + h->classes[ci].n <= pos[k]) ++ci;
        const ClassInfo& src = h->classes[ci];
        int64_t q = k;
        while (q < n_sel && pos[q] < src.first + src.n) ++q;
        ClassInfo c{};
        c.first = k;
        c.n = (int32_t)(q - k);
        c.n_pad = (int32_t)((c.n + kPadItems - 1) / kPadItems * kPadItems);
        c.r = src.r;
        c.W = src.W;
        c.word_off = word_off;
        word_off += (int64_t)c.W * c.n_pad;
        sel->classes.push_back(c);
        src_class.push_back((int)ci);
        k = q;
    }
    BM_TRY(ensure(&h->sel_arena_d, &h->sel_arena_cap, std::max<int64_t>(word_off, 1), st));
    BM_TRY(ensure(&h->sel_idx_d, &h->sel_idx_cap, std::max<int64_t>(3 * n_sel, 3), st));
    int32_t* sel2pos = h->sel_idx_d;
    int32_t* sel2orig = h->sel_idx_d + n_sel;
    int32_t* fsel = h->sel_idx_d + 2 * n_sel;
    if (n_sel) {
        BM_CUDA(cudaMemcpyAsync(sel2pos, pos.data(), n_sel * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        k_gather_meta<<<(unsigned)((n_sel + 255) / 256), 256, 0, st>>>(sel2pos, n_sel, h->pos2orig_d, h->f_d,
                                                                      sel2orig, fsel);
    }
    for (size_t a = 0; a < sel->classes.size(); ++a) {
        const ClassInfo& c = sel->classes[a];
        const ClassInfo& src = h->classes[src_class[a]];
        const int64_t cnt = (int64_t)c.W * c.n_pad;
        k_gather_cols<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(h->arena_d, src.word_off, src.n_pad, src.first,
                                                                     sel2pos, c.first, c.n, c.n_pad, c.W,
                                                                     h->sel_arena_d + c.word_off);
    }
    BM_CUDA(cudaGetLastError());
    BM_CUDA(cudaStreamSynchronize(st));  // `pos` (host) must outlive the H2D copy
    sel->arena = h->sel_arena_d;
    sel->f = fsel;
    sel->sel2pos = sel2pos;
    sel->sel2orig = sel2orig;
    return BATMAP_OK;
}

}  // namespace bm
