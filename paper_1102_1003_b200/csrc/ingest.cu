// ingest.cu -- NEXT-3: FIMI-repository text -> vertical tidlists on the device, and the
// frequent-item pre-filter.
//
// What ("taken from the Frequent Itemset Mining Dataset Repository"; SPEC S:504-512;
// readings #21-#25 of DESIGN.md): one transaction per line, 0-based line index = tid (reading
// #2), decimal item labels separated by spaces / tabs / '\r'; duplicates within a line collapse;
// blank lines are empty transactions; labels are re-densified in ascending order with the map
// kept; any other byte (or a label > 2^32 - 1) is an error reported with its 1-based line.  The
// vertical layout is what batmap_build consumes.  The pre-filter keeps the items whose
// support |S_i| reaches the threshold (the paper assumes infrequent items removed; no
// pair containing one can reach the threshold).
//
// How (B200): the text is read in 4 KB blocks (16 bytes per thread, 128-bit loads).  Pass 1
// counts token starts and newlines per block; a device scan turns them into per-block bases;
// pass 2 re-walks each thread's bytes with a block scan for its own bases, parses each token
// and writes one 64-bit key (label << tid_bits | tid) in text order.  A stable CUB radix sort over
// the label bits only (the keys already ascend in tid), a unique (duplicates within a line), a
// flag-and-scan of label changes and one emit
// kernel produce offsets / tids / labels.  Three host synchronisations in total (token count,
// max label and error position, item count); everything else is stream-ordered.
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

#include "fimi.h"

namespace bm {

constexpr int kIngThreads = 256;
constexpr int kIngBytes = 16;                          // bytes per thread
constexpr int kIngBlock = kIngThreads * kIngBytes;     // bytes per block

__device__ __forceinline__ bool is_digit(uint32_t c) { return c - 48u < 10u; }
__device__ __forceinline__ bool is_blank(uint32_t c) { return c == 32u || c == 9u || c == 13u; }

// 16 bytes at pos (bytes at or beyond n read as ' ')
__device__ __forceinline__ void load16(const uint8_t* __restrict__ text, int64_t n, int64_t pos, bool aligned,
                                       uint8_t (&b)[kIngBytes]) {
    if (aligned && pos + kIngBytes <= n) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(text + pos));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < kIngBytes; ++k) b[k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
    } else {
#pragma unroll
        for (int k = 0; k < kIngBytes; ++k) b[k] = pos + k < n ? __ldg(text + pos + k) : (uint8_t)32;
    }
}

struct Counts {
    int tok, nl;
};

__device__ __forceinline__ Counts count16(const uint8_t* __restrict__ text, int64_t n, int64_t pos, bool aligned,
                                          uint8_t (&b)[kIngBytes], unsigned long long* err_pos) {
    load16(text, n, pos, aligned, b);
    uint32_t prev = (pos > 0 && pos <= n) ? __ldg(text + pos - 1) : 32u;  // threads past the end read nothing
    Counts c{0, 0};
#pragma unroll
    for (int k = 0; k < kIngBytes; ++k) {
        const uint32_t ch = b[k];
        const bool d = is_digit(ch);
        c.tok += d && !is_digit(prev);
        c.nl += ch == 10u;
        if (!d && ch != 10u && !is_blank(ch) && err_pos) atomicMin(err_pos, (unsigned long long)(pos + k));
        prev = ch;
    }
    return c;
}

__global__ void __launch_bounds__(kIngThreads) k_fimi_count(const uint8_t* __restrict__ text, int64_t n, bool aligned,
                                                            int64_t* __restrict__ blk_tok, int64_t* __restrict__ blk_nl,
                                                            unsigned long long* __restrict__ err_pos) {
    using BR = cub::BlockReduce<int, kIngThreads>;
    __shared__ typename BR::TempStorage t1, t2;
    uint8_t b[kIngBytes];
    const int64_t pos = (int64_t)blockIdx.x * kIngBlock + (int64_t)threadIdx.x * kIngBytes;
    const Counts c = count16(text, n, pos, aligned, b, err_pos);
    const int tok = BR(t1).Sum(c.tok);
    const int nl = BR(t2).Sum(c.nl);
    if (threadIdx.x == 0) {
        blk_tok[blockIdx.x] = tok;
        blk_nl[blockIdx.x] = nl;
    }
}

__global__ void __launch_bounds__(kIngThreads) k_fimi_keys(const uint8_t* __restrict__ text, int64_t n, bool aligned,
                                                           const int64_t* __restrict__ tok_base,
                                                           const int64_t* __restrict__ nl_base, int tid_bits,
                                                           uint64_t* __restrict__ keys,
                                                           unsigned int* __restrict__ max_label,
                                                           unsigned long long* __restrict__ err_pos) {
    using BS = cub::BlockScan<int, kIngThreads>;
    __shared__ typename BS::TempStorage t1, t2;
    uint8_t b[kIngBytes];
    const int64_t pos = (int64_t)blockIdx.x * kIngBlock + (int64_t)threadIdx.x * kIngBytes;
    const Counts c = count16(text, n, pos, aligned, b, nullptr);
    int tok_ex, nl_ex;
    BS(t1).ExclusiveSum(c.tok, tok_ex);
    BS(t2).ExclusiveSum(c.nl, nl_ex);
    int64_t tok = tok_base[blockIdx.x] + tok_ex;
    int64_t line = nl_base[blockIdx.x] + nl_ex;
    unsigned int mx = 0;
    // a token is parsed from the registers while it lies in this thread's 16 bytes; digits that
    // continue a token from the previous thread's bytes belong to that thread (it reads on)
    bool skipping = pos > 0 && pos <= n && is_digit(__ldg(text + pos - 1));
    bool in = false, ovf = false;
    uint64_t v = 0;
    int64_t start = 0;
    auto emit = [&]() {
        if (ovf) {
            atomicMin(err_pos, (unsigned long long)start);
            v = 0;
        }
        keys[tok++] = (v << tid_bits) | (uint64_t)line;
        mx = max(mx, (unsigned int)v);
    };
#pragma unroll
    for (int k = 0; k < kIngBytes; ++k) {
        const uint32_t ch = b[k];
        const bool d = is_digit(ch);
        if (skipping) {
            if (d) continue;
            skipping = false;
        }
        if (d) {
            if (!in) {
                in = true;
                ovf = false;
                v = 0;
                start = pos + k;
            }
            v = v * 10u + (ch - 48u);
            ovf |= v > 0xFFFFFFFFull;
            if (ovf) v = 0xFFFFFFFFull + 1;  // saturate (no wrap on very long digit runs)
        } else {
            if (in) {
                emit();
                in = false;
            }
            line += ch == 10u;
        }
    }
    if (in) {  // the token runs past this thread's bytes
        for (int64_t q = pos + kIngBytes; q < n; ++q) {
            const uint32_t d = __ldg(text + q);
            if (!is_digit(d)) break;
            v = v * 10u + (d - 48u);
            ovf |= v > 0xFFFFFFFFull;
            if (ovf) v = 0xFFFFFFFFull + 1;
        }
        emit();
    }
    mx = __reduce_max_sync(0xFFFFFFFFu, mx);  // one atomic per warp
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_label, mx);
}

// Line (1-based) of byte position p: newlines before the block of p plus those in it before p.
__global__ void k_fimi_line_of(const uint8_t* __restrict__ text, const int64_t* __restrict__ nl_base,
                               const unsigned long long* __restrict__ err_pos, int64_t* __restrict__ line_out) {
    using BR = cub::BlockReduce<int, kIngThreads>;
    __shared__ typename BR::TempStorage t;
    const int64_t p = (int64_t)*err_pos;
    const int64_t blk = p / kIngBlock;
    int c = 0;
    for (int64_t q = blk * kIngBlock + threadIdx.x; q < p; q += kIngThreads) c += __ldg(text + q) == 10u;
    const int s = BR(t).Sum(c);
    if (threadIdx.x == 0) *line_out = nl_base[blk] + s + 1;
}

__global__ void k_fimi_flags(const uint64_t* __restrict__ keys, int64_t nnz, int tid_bits, int32_t* __restrict__ flag) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    flag[k] = (k == 0 || (keys[k] >> tid_bits) != (keys[k - 1] >> tid_bits)) ? 1 : 0;
}

__global__ void k_fimi_emit(const uint64_t* __restrict__ keys, const int32_t* __restrict__ flag,
                            const int32_t* __restrict__ dense, int64_t nnz, int tid_bits, int32_t* __restrict__ tids,
                            int64_t* __restrict__ off, uint32_t* __restrict__ labels) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const uint64_t key = keys[k];
    tids[k] = (int32_t)(key & ((uint64_t(1) << tid_bits) - 1));
    if (flag[k]) {
        const int32_t d = dense[k];
        labels[d] = (uint32_t)(key >> tid_bits);
        off[d] = k;
    }
}

// Frequent-item filter: keep item i iff offsets[i+1] - offsets[i] >= thr.
struct SupportAtLeast {
    const int64_t* off;
    int64_t thr;
    __host__ __device__ __forceinline__ bool operator()(const int32_t& i) const { return off[i + 1] - off[i] >= thr; }
};

__global__ void k_gather_sizes(const int64_t* __restrict__ off, const int32_t* __restrict__ items, int64_t n_sel,
                               int64_t* __restrict__ sizes) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n_sel) sizes[k] = off[items[k] + 1] - off[items[k]];
}

// one thread per output element: binary search of its kept item in new_off (balanced for Zipf
// list lengths); the first element of each list also moves the label
__global__ void k_gather_lists(const int64_t* __restrict__ off, const int32_t* __restrict__ tids,
                               const uint32_t* __restrict__ labels, const int32_t* __restrict__ items, int64_t n_sel,
                               const int64_t* __restrict__ new_off, int64_t nnz, int32_t* __restrict__ new_tids,
                               uint32_t* __restrict__ new_labels) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n_sel - 1;  // last k with new_off[k] <= e
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (__ldg(new_off + mid) <= e) lo = mid;
            else hi = mid - 1;
        }
        const int32_t i = __ldg(items + lo);
        new_tids[e] = __ldg(tids + __ldg(off + i) + (e - __ldg(new_off + lo)));
    }
    if (labels)
        for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_sel; k += (int64_t)gridDim.x * blockDim.x)
            new_labels[k] = labels[items[k]];
}

static int bits_for(uint64_t v) {  // bits needed to represent 0..v
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

static batmap_status cub_run(void** tmp, size_t* cap, size_t need, cudaStream_t st) {
    if (need <= *cap) return BATMAP_OK;
    dfree(*tmp, st);
    *tmp = nullptr;
    *cap = 0;
    BM_TRY(dalloc(tmp, need, st));
    *cap = need;
    return BATMAP_OK;
}

batmap_status fimi_parse(const uint8_t* text, int64_t n, cudaStream_t st, batmap_fimi* h, int64_t* bad_line) {
    *bad_line = -1;
    if (n == 0) {
        BM_TRY(dalloc_t(&h->off_d, 1, st));
        BM_CUDA(cudaMemsetAsync(h->off_d, 0, sizeof(int64_t), st));
        BM_TRY(dalloc_t(&h->tids_d, 1, st));
        BM_TRY(dalloc_t(&h->labels_d, 1, st));
        return BATMAP_OK;
    }
    const bool aligned = ((uintptr_t)text & 15) == 0;
    const int64_t nb = (n + kIngBlock - 1) / kIngBlock;
    if (nb > INT32_MAX) {
        set_error("text of %lld bytes is too large", (long long)n);
        return BATMAP_E_OVERFLOW;
    }
    void* tmp = nullptr;
    size_t tmp_cap = 0;
    int64_t *blk_tok = nullptr, *blk_nl = nullptr, *scal = nullptr;
    unsigned long long* err_pos = nullptr;
    unsigned int* max_label = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    int32_t *flag = nullptr, *dense = nullptr;
    int64_t* nsel_d = nullptr;
    batmap_status rc = BATMAP_OK;
    auto cleanup = [&]() {
        dfree(tmp, st);
        dfree(blk_tok, st);
        dfree(blk_nl, st);
        dfree(scal, st);
        dfree(err_pos, st);
        dfree(max_label, st);
        dfree(keys, st);
        dfree(keys2, st);
        dfree(flag, st);
        dfree(dense, st);
        dfree(nsel_d, st);
    };
#define ING_TRY(expr)              \
    do {                           \
        rc = (expr);               \
        if (rc != BATMAP_OK) {     \
            cleanup();             \
            return rc;             \
        }                          \
    } while (0)
#define ING_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            set_error("%s:%d %s -> %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
            cleanup();                                                                   \
            return BATMAP_E_CUDA;                                                        \
        }                                                                                \
    } while (0)
    ING_TRY(dalloc_t(&blk_tok, nb + 1, st));
    ING_TRY(dalloc_t(&blk_nl, nb + 1, st));
    ING_TRY(dalloc_t(&scal, 4, st));
    ING_TRY(dalloc_t(&err_pos, 1, st));
    ING_TRY(dalloc_t(&max_label, 1, st));
    ING_CUDA(cudaMemsetAsync(err_pos, 0xFF, sizeof(unsigned long long), st));
    ING_CUDA(cudaMemsetAsync(max_label, 0, sizeof(unsigned int), st));
    ING_CUDA(cudaMemsetAsync(blk_tok + nb, 0, sizeof(int64_t), st));
    ING_CUDA(cudaMemsetAsync(blk_nl + nb, 0, sizeof(int64_t), st));
    k_fimi_count<<<(unsigned)nb, kIngThreads, 0, st>>>(text, n, aligned, blk_tok, blk_nl, err_pos);
    ING_CUDA(cudaGetLastError());
    // exclusive sums over nb + 1 entries: entry nb = the totals
    size_t need = 0;
    ING_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, blk_tok, blk_tok, nb + 1, st));
    ING_TRY(cub_run(&tmp, &tmp_cap, need, st));
    ING_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, blk_tok, blk_tok, nb + 1, st));
    ING_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, blk_nl, blk_nl, nb + 1, st));
    int64_t tot[2];
    uint8_t last = 0;
    ING_CUDA(cudaMemcpyAsync(&tot[0], blk_tok + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    ING_CUDA(cudaMemcpyAsync(&tot[1], blk_nl + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    ING_CUDA(cudaMemcpyAsync(&last, text + n - 1, 1, cudaMemcpyDeviceToHost, st));
    ING_CUDA(cudaStreamSynchronize(st));  // sync 1: token count, transaction count
    const int64_t T = tot[0];
    const int64_t m = tot[1] + (last != 10 ? 1 : 0);
    if (m >= (int64_t(1) << 31)) {
        set_error("%lld transactions >= 2^31", (long long)m);
        cleanup();
        return BATMAP_E_OVERFLOW;
    }
    const int tid_bits = std::max(1, bits_for((uint64_t)(m > 0 ? m - 1 : 0)));
    ING_TRY(dalloc_t(&keys, T, st));
    ING_TRY(dalloc_t(&keys2, T, st));
    k_fimi_keys<<<(unsigned)nb, kIngThreads, 0, st>>>(text, n, aligned, blk_tok, blk_nl, tid_bits, keys, max_label,
                                                     err_pos);
    ING_CUDA(cudaGetLastError());
    unsigned long long ep = 0;
    unsigned int mx = 0;
    ING_CUDA(cudaMemcpyAsync(&ep, err_pos, sizeof(ep), cudaMemcpyDeviceToHost, st));
    ING_CUDA(cudaMemcpyAsync(&mx, max_label, sizeof(mx), cudaMemcpyDeviceToHost, st));
    ING_CUDA(cudaStreamSynchronize(st));  // sync 2: errors, key width
    if (ep != ~0ull) {
        k_fimi_line_of<<<1, kIngThreads, 0, st>>>(text, blk_nl, err_pos, scal);
        int64_t ln = -1;
        ING_CUDA(cudaMemcpyAsync(&ln, scal, sizeof(ln), cudaMemcpyDeviceToHost, st));
        ING_CUDA(cudaStreamSynchronize(st));
        *bad_line = ln;
        set_error("line %lld: invalid byte or item id > 2^32 - 1", (long long)ln);
        cleanup();
        return BATMAP_E_INVALID;
    }
    const int end_bit = tid_bits + std::max(1, bits_for(mx));
    int64_t nnz = 0;
    if (T > 0) {
        // keys are written in text order, i.e. ascending tid; the (stable, LSD) radix sort therefore
        // only needs the label bits [tid_bits, end_bit) to order by (label, tid)
        ING_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, need, keys, keys2, T, tid_bits, end_bit, st));
        ING_TRY(cub_run(&tmp, &tmp_cap, need, st));
        ING_CUDA(cub::DeviceRadixSort::SortKeys(tmp, need, keys, keys2, T, tid_bits, end_bit, st));
        ING_TRY(dalloc_t(&nsel_d, 1, st));
        ING_CUDA(cub::DeviceSelect::Unique(nullptr, need, keys2, keys, nsel_d, T, st));
        ING_TRY(cub_run(&tmp, &tmp_cap, need, st));
        ING_CUDA(cub::DeviceSelect::Unique(tmp, need, keys2, keys, nsel_d, T, st));
        ING_CUDA(cudaMemcpyAsync(&nnz, nsel_d, sizeof(nnz), cudaMemcpyDeviceToHost, st));
        ING_CUDA(cudaStreamSynchronize(st));  // sync 3: nnz
    }
    ING_TRY(dalloc_t(&h->tids_d, nnz, st));
    ING_TRY(dalloc_t(&h->off_d, nnz + 1, st));  // n_items <= nnz
    ING_TRY(dalloc_t(&h->labels_d, nnz, st));
    int64_t n_items = 0;
    if (nnz > 0) {
        ING_TRY(dalloc_t(&flag, nnz, st));
        ING_TRY(dalloc_t(&dense, nnz, st));
        const unsigned g = (unsigned)((nnz + 255) / 256);
        k_fimi_flags<<<g, 256, 0, st>>>(keys, nnz, tid_bits, flag);
        ING_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, flag, dense, nnz, st));
        ING_TRY(cub_run(&tmp, &tmp_cap, need, st));
        ING_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, flag, dense, nnz, st));
        k_fimi_emit<<<g, 256, 0, st>>>(keys, flag, dense, nnz, tid_bits, h->tids_d, h->off_d, h->labels_d);
        ING_CUDA(cudaGetLastError());
        int32_t lf[2];
        ING_CUDA(cudaMemcpyAsync(&lf[0], dense + nnz - 1, 4, cudaMemcpyDeviceToHost, st));
        ING_CUDA(cudaMemcpyAsync(&lf[1], flag + nnz - 1, 4, cudaMemcpyDeviceToHost, st));
        ING_CUDA(cudaStreamSynchronize(st));
        n_items = (int64_t)lf[0] + lf[1];
    }
    ING_CUDA(cudaMemcpyAsync(h->off_d + n_items, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    ING_CUDA(cudaStreamSynchronize(st));  // nnz is a host local
    h->n_items = n_items;
    h->nnz = nnz;
    h->m = m;
    cleanup();
    return BATMAP_OK;
#undef ING_TRY
#undef ING_CUDA
}

batmap_status frequent_items(const int64_t* off, int64_t n_items, uint32_t min_support, int32_t* items_out,
                             int64_t* n_out, cudaStream_t st) {
    *n_out = 0;
    if (n_items == 0) return BATMAP_OK;
    int64_t* cnt_d = nullptr;
    void* tmp = nullptr;
    size_t need = 0;
    cub::CountingInputIterator<int32_t> it(0);
    const SupportAtLeast pred{off, (int64_t)min_support};
    BM_CUDA(cub::DeviceSelect::If(nullptr, need, it, items_out, (int64_t*)nullptr, n_items, pred, st));
    BM_TRY(dalloc(&tmp, need, st));
    batmap_status rc = dalloc_t(&cnt_d, 1, st);
    if (rc == BATMAP_OK) {
        cudaError_t e = cub::DeviceSelect::If(tmp, need, it, items_out, cnt_d, n_items, pred, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(n_out, cnt_d, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            set_error("frequent_items: %s", cudaGetErrorString(e));
            rc = BATMAP_E_CUDA;
        }
    }
    dfree(tmp, st);
    dfree(cnt_d, st);
    return rc;
}

batmap_status fimi_filter(batmap_fimi* h, uint32_t min_support, cudaStream_t st) {
    if (h->n_items == 0) return BATMAP_OK;
    int32_t* items = nullptr;
    int64_t *sizes = nullptr, *new_off = nullptr;
    int32_t* new_tids = nullptr;
    uint32_t* new_labels = nullptr;
    void* tmp = nullptr;
    int64_t n_sel = 0;
    BM_TRY(dalloc_t(&items, h->n_items, st));
    batmap_status rc = frequent_items(h->off_d, h->n_items, min_support, items, &n_sel, st);
    if (rc != BATMAP_OK) {
        dfree(items, st);
        return rc;
    }
    auto fail = [&](batmap_status r) {
        dfree(items, st);
        dfree(sizes, st);
        dfree(new_off, st);
        dfree(new_tids, st);
        dfree(new_labels, st);
        dfree(tmp, st);
        return r;
    };
    if ((rc = dalloc_t(&sizes, n_sel + 1, st)) != BATMAP_OK) return fail(rc);
    if ((rc = dalloc_t(&new_off, n_sel + 1, st)) != BATMAP_OK) return fail(rc);
    if (cudaMemsetAsync(sizes + n_sel, 0, sizeof(int64_t), st) != cudaSuccess) return fail(BATMAP_E_CUDA);
    if (n_sel) k_gather_sizes<<<(unsigned)((n_sel + 255) / 256), 256, 0, st>>>(h->off_d, items, n_sel, sizes);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, sizes, new_off, n_sel + 1, st);
    if ((rc = dalloc(&tmp, need, st)) != BATMAP_OK) return fail(rc);
    if (cub::DeviceScan::ExclusiveSum(tmp, need, sizes, new_off, n_sel + 1, st) != cudaSuccess)
        return fail(BATMAP_E_CUDA);
    int64_t nnz = 0;
    if (cudaMemcpyAsync(&nnz, new_off + n_sel, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return fail(BATMAP_E_CUDA);
    if ((rc = dalloc_t(&new_tids, nnz, st)) != BATMAP_OK) return fail(rc);
    if ((rc = dalloc_t(&new_labels, n_sel, st)) != BATMAP_OK) return fail(rc);
    if (n_sel) {
        const int64_t work = std::max(nnz, n_sel);
        const unsigned g = (unsigned)std::min<int64_t>((work + 255) / 256, 148 * 16);
        k_gather_lists<<<g, 256, 0, st>>>(h->off_d, h->tids_d, h->labels_d, items, n_sel, new_off, nnz, new_tids,
                                          new_labels);
    }
    if (cudaGetLastError() != cudaSuccess) return fail(BATMAP_E_CUDA);
    dfree(h->off_d, st);
    dfree(h->tids_d, st);
    dfree(h->labels_d, st);
    h->off_d = new_off;
    h->tids_d = new_tids;
    h->labels_d = new_labels;
    h->n_items = n_sel;
    h->nnz = nnz;
    new_off = nullptr;
    new_tids = nullptr;
    new_labels = nullptr;
    return fail(BATMAP_OK);
}

// The vertical database restricted to `items` (in the given order): offsets_out [n_sel + 1] and,
// when it fits, tids_out; *nnz_out = the selected entries.  One synchronisation (the size).
batmap_status select_csr(const int64_t* off, const int32_t* tids, const int32_t* items, int64_t n_sel,
                         int64_t* offsets_out, int32_t* tids_out, int64_t tids_capacity, int64_t* nnz_out,
                         cudaStream_t st) {
    int64_t* sizes = nullptr;
    void* tmp = nullptr;
    BM_TRY(dalloc_t(&sizes, n_sel + 1, st));
    batmap_status rc = BATMAP_OK;
    size_t need = 0;
    if (cudaMemsetAsync(sizes + n_sel, 0, sizeof(int64_t), st) != cudaSuccess) rc = BATMAP_E_CUDA;
    if (rc == BATMAP_OK && n_sel)
        k_gather_sizes<<<(unsigned)((n_sel + 255) / 256), 256, 0, st>>>(off, items, n_sel, sizes);
    if (rc == BATMAP_OK) {
        cub::DeviceScan::ExclusiveSum(nullptr, need, sizes, offsets_out, n_sel + 1, st);
        rc = dalloc(&tmp, need, st);
    }
    if (rc == BATMAP_OK && cub::DeviceScan::ExclusiveSum(tmp, need, sizes, offsets_out, n_sel + 1, st) != cudaSuccess)
        rc = BATMAP_E_CUDA;
    int64_t nnz = 0;
    if (rc == BATMAP_OK &&
        (cudaMemcpyAsync(&nnz, offsets_out + n_sel, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
         cudaStreamSynchronize(st) != cudaSuccess))
        rc = BATMAP_E_CUDA;
    dfree(sizes, st);
    dfree(tmp, st);
    if (rc != BATMAP_OK) {
        set_error("select_csr: %s", cudaGetErrorString(cudaGetLastError()));
        return rc;
    }
    *nnz_out = nnz;
    if (nnz > tids_capacity) {
        set_error("capacity %lld < %lld tids", (long long)tids_capacity, (long long)nnz);
        return BATMAP_E_CAPACITY;
    }
    if (n_sel && nnz) {
        const unsigned g = (unsigned)std::min<int64_t>((nnz + 255) / 256, 148 * 16);
        k_gather_lists<<<g, 256, 0, st>>>(off, tids, nullptr, items, n_sel, offsets_out, nnz, tids_out, nullptr);
        BM_CUDA(cudaGetLastError());
    }
    return BATMAP_OK;
}

}  // namespace bm
