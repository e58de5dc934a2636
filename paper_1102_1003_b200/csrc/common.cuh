// common.cuh -- shared definitions of the CUDA path (never shared with oracle/).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/batmap.h"

namespace bm {

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
const char* get_error();

struct Status {
    batmap_status code = BATMAP_OK;
};

#define BM_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) {                                                             \
            ::bm::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
            return (e_ == cudaErrorMemoryAllocation) ? BATMAP_E_NOMEM : BATMAP_E_CUDA;       \
        }                                                                                    \
    } while (0)

#define BM_TRY(expr)                        \
    do {                                    \
        batmap_status s_ = (expr);          \
        if (s_ != BATMAP_OK) return s_;     \
    } while (0)

// ------------------------------------------------------------------ π_t (reading #3)
// Seeded bijection of [0, U), U = 127 * 2^s: four rounds of {v *= k (mod 2^w); v ^= v >> ceil(w/2)}
// on w = s + 7 bits, cycle-walked into [0, U).  Optional table override (test hook).
struct PiParams {
    uint32_t s, w, U, mask, half;
    uint32_t key[3][4];
    uint32_t kinv[3][4];    // key^-1 mod 2^w (the byte-table build inverts π, reading #3)
    const uint32_t* table;  // device [3][U] or nullptr
};

__host__ __device__ __forceinline__ uint32_t pi_key(const PiParams& P, int t, int r) {
    // select instead of a dynamic index (keeps the parameter struct out of local memory)
    return t == 0 ? P.key[0][r] : (t == 1 ? P.key[1][r] : P.key[2][r]);
}

__host__ __device__ __forceinline__ uint32_t pi_mix(const PiParams& P, int t, uint32_t v) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        v = (v * pi_key(P, t, r)) & P.mask;
        v ^= v >> P.half;
    }
    return v;
}

__host__ __device__ __forceinline__ uint32_t pi_kinv(const PiParams& P, int t, int r) {
    return t == 0 ? P.kinv[0][r] : (t == 1 ? P.kinv[1][r] : P.kinv[2][r]);
}

// mix^-1: the rounds in reverse order; v ^= v >> half is an involution on w bits (half >= w/2)
__host__ __device__ __forceinline__ uint32_t pi_unmix(const PiParams& P, int t, uint32_t v) {
#pragma unroll
    for (int r = 3; r >= 0; --r) {
        v ^= v >> P.half;
        v = (v * pi_kinv(P, t, r)) & P.mask;
    }
    return v;
}

// π_t^-1 on [0, U): walk mix^-1 back until the value is in [0, U) again (the cycle-walk's inverse:
// every value strictly between x and π_t(x) on x's mix orbit is >= U).  Hash form only (P.table
// == nullptr).
__device__ __forceinline__ uint32_t pi_inverse(const PiParams& P, int t, uint32_t v) {
    uint32_t x = pi_unmix(P, t, v);
    while (x >= P.U) x = pi_unmix(P, t, x);
    return x;
}

// t is 0-based (table t+1 of the paper)
__device__ __forceinline__ uint32_t pi_eval(const PiParams& P, int t, uint32_t x) {
    if (P.table) return __ldg(P.table + (size_t)t * P.U + x);
    uint32_t v = pi_mix(P, t, x);
    while (v >= P.U) v = pi_mix(P, t, v);
    return v;
}

PiParams make_pi(uint64_t seed, int s, const uint32_t* table);

// h_t(x) = 3 r0 floor((v mod r)/r0) + (v mod r0) + (t-1) r0,  v = π_t(x).
// t 0-based here; r, r0 powers of two.
__host__ __device__ __forceinline__ uint32_t slot_of(int t, uint32_t v, uint32_t r, uint32_t r0,
                                                     int log2r0) {
    uint32_t vr = v & (r - 1);
    return 3u * r0 * (vr >> log2r0) + (v & (r0 - 1)) + (uint32_t)t * r0;
}

constexpr uint32_t kEmpty = 0xFFFFFFFFu;    // working-table ⊥ (tids < 2^31)
constexpr uint8_t kNullByte = 0x7F;          // encoded ⊥ (reading #1)
constexpr uint32_t kNullWord = 0x7F7F7F7Fu;

// ------------------------------------------------------------------ layout
// Items are sorted by width into classes of equal r.  Class a stores its BatMaps
// word-major: word w of the item at column c (0 <= c < n_pad) is
//   arena[word_off + (int64)w * n_pad + c];  padding columns hold ⊥ words.
constexpr int kPadItems = 128;

struct ClassInfo {
    int64_t first;     // first position (in width-sorted order) of this class
    int64_t word_off;  // offset of the class block in the arena (words)
    int32_t n;         // items in class
    int32_t n_pad;     // n rounded up to kPadItems
    int32_t r;         // table range
    int32_t W;         // words per BatMap = 3r/4
};

struct Cand {
    uint32_t i, j, c;  // selection indices (width-sorted) and raw count
};

// K2 launch description of one selection (full collection or a subset of items)
struct Selection {
    std::vector<ClassInfo> classes;
    const uint32_t* arena = nullptr;  // device
    const int32_t* f = nullptr;       // device, per selection index: failure counts
    const int32_t* sel2pos = nullptr; // device or nullptr (identity)
    const int32_t* sel2orig = nullptr;// device
    int64_t n_sel = 0;
};

}  // namespace bm

namespace bm {
struct K2Prepared;
}

struct batmap_collection {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;

    int64_t n = 0, m = 0;
    int64_t nnz = 0;  // entries of the input CSR (set by the build)
    int s = 0;
    int64_t U = 0;
    int64_t r0 = 0;
    int log2r0 = 0;
    uint64_t seed = 0;
    uint32_t r_min = 128, max_loop_opt = 0;
    bm::PiParams pi{};

    std::vector<int32_t> pos2orig_h, orig2pos_h;
    std::vector<int32_t> size_orig_h;  // |S_i| by caller id (the frequent-item filter)
    std::vector<bm::ClassInfo> classes;
    int64_t arena_bytes_raw = 0;  // sum 3 r_i
    int64_t arena_words = 0;      // incl. padding

    int32_t* pos2orig_d = nullptr;
    int32_t* orig2pos_d = nullptr;
    uint32_t* arena_d = nullptr;
    int32_t* f_d = nullptr;  // failures per position

    // failure list F, by position, tids ascending
    int64_t n_fail = 0;
    int64_t* fail_off_d = nullptr;  // n+1
    int32_t* fail_tid_d = nullptr;  // n_fail
    // A_b for failed transactions b: fidx_of_tid[b] = k or -1; ab_pos[ab_off[k]..ab_off[k+1])
    int64_t n_ftid = 0;
    int32_t* fidx_of_tid_d = nullptr;  // m
    int64_t* ab_off_d = nullptr;       // n_ftid + 1
    int32_t* ab_pos_d = nullptr;

    // pair-phase scratch (grown on demand)
    bm::Cand* cand_d = nullptr;
    int64_t cand_cap = 0;
    unsigned long long* ctr_d = nullptr;  // [0] candidates, [1] emitted
    uint64_t* key_d = nullptr;            // sort keys / values, 2 buffers each
    uint32_t* val_d = nullptr;
    int64_t kv_cap = 0;
    void* cub_tmp = nullptr;
    size_t cub_tmp_bytes = 0;
    // K2: plan of the full selection prepared during the build; counters of accumulated rectangles
    bm::K2Prepared* k2prep = nullptr;
    // sharded build (batmap_build_shard): this part's failure records until batmap_shard_import
    bool shard_pending = false;
    int shard_part = 0, shard_n_parts = 1;
    std::vector<int32_t> shard_rot;  // per class: part p builds column chunk (p + shard_rot[a]) mod N
    uint64_t* shard_fails_d = nullptr;
    int64_t shard_n_fail = 0;
    uint32_t* cnt_d = nullptr;
    int64_t cnt_cap = 0;
    uint32_t* tail_d = nullptr;  // partial counts of the cut tail tiles (k2_tiled -> k2_tail_threshold)
    int64_t tail_cap = 0;
    // selection scratch
    uint32_t* sel_arena_d = nullptr;
    int64_t sel_arena_cap = 0;
    int32_t* sel_idx_d = nullptr;  // [0..cap): sel2pos, [cap..2cap): sel2orig, [2cap..3cap): f_sel
    int64_t sel_idx_cap = 0;

    // phase timing (CUDA events on the launching stream), evaluated lazily by batmap_stats
    cudaEvent_t ev[12] = {};
    bool ev_ok = false;
    bool build_timed = false, pairs_timed = false;
    batmap_stats_t stats{};
    int64_t launches = 0;  // running count of kernels launched by this handle

    // result cache for the two-call capacity protocol
    batmap_triple* res_d = nullptr;
    int64_t res_cap = 0;
    int64_t res_n = -1;
    const int32_t* res_items = nullptr;
    int64_t res_nsel = -1;
    uint32_t res_thr = 0, res_flags = 0;
    int32_t res_part = -1, res_nparts = -1;
};

namespace bm {
// event slots: 0/1 build, 2/3 K1 insert, 4/5 K1 encode, 6/7 pairs, 8/9 K2, 10 K3 start (K3 ends at 7)
enum { EV_B0 = 0, EV_B1, EV_I0, EV_I1, EV_E0, EV_E1, EV_P0, EV_P1, EV_K20, EV_K21, EV_K30, EV_COUNT };
inline void rec(batmap_collection* h, int idx, cudaStream_t st) {
    if (!h->ev_ok) {
        h->ev_ok = true;
        for (int i = 0; i < EV_COUNT; ++i)
            if (cudaEventCreate(&h->ev[i]) != cudaSuccess) h->ev_ok = false;
        if (!h->ev_ok) cudaGetLastError();
    }
    if (h->ev_ok) cudaEventRecord(h->ev[idx], st);
}
// allocation helpers (stream-ordered pool)
batmap_status dalloc(void** p, size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);
// per-thread pinned staging buffers: slot 0 for the build's host tables, slot 1 for the K2 plan
// upload (both reused by the next call of the thread, after its stream synchronisation)
void* host_staging(size_t bytes, int slot = 0);
// tids may be NULL exactly when the tidlists are all empty (a zero-length int32[offsets[n]]): reads
// offsets[n_items] (device) when tids is NULL and n_items > 0; E_INVALID if it is not 0.
batmap_status check_tids_device(const int64_t* offsets, const int32_t* tids, int64_t n_items, cudaStream_t st);
// k scalar device -> host copies (each <= 8 bytes) then one synchronisation of st
batmap_status read_scalars(cudaStream_t st, int k, const void* const* src, const size_t* bytes, void* const* dst);
template <typename T>
batmap_status read_scalar(cudaStream_t st, const T* src, T* dst) {
    const void* s[1] = {src};
    const size_t b[1] = {sizeof(T)};
    void* d[1] = {dst};
    return read_scalars(st, 1, s, b, d);
}
template <typename T>
batmap_status dalloc_t(T** p, int64_t count, cudaStream_t s) {
    return dalloc(reinterpret_cast<void**>(p), (size_t)(count > 0 ? count : 1) * sizeof(T), s);
}
// Frees a function's scratch buffers on every return path, early error returns included
// (stream-ordered; each registered pointer is freed once and reset to nullptr).
class Scratch {
  public:
    explicit Scratch(cudaStream_t s) : st_(s) {}
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    template <typename T>
    void own(T** p) {
        slots_[n_++] = reinterpret_cast<void**>(p);
    }
    ~Scratch() {
        for (int i = 0; i < n_; ++i) {
            dfree(*slots_[i], st_);
            *slots_[i] = nullptr;
        }
    }

  private:
    cudaStream_t st_;
    void** slots_[16];
    int n_ = 0;
};
template <typename T>
batmap_status ensure(T** p, int64_t* cap, int64_t need, cudaStream_t s) {
    if (*p && *cap >= need) return BATMAP_OK;
    if (*p) dfree(*p, s);
    *p = nullptr;
    int64_t c = need > 1024 ? need + need / 4 : 1024;
    BM_TRY(dalloc_t(p, c, s));
    *cap = c;
    return BATMAP_OK;
}

// build.cu
batmap_status build_collection(batmap_collection* h, const int64_t* offsets, const int32_t* tids,
                               const batmap_build_opts* o, int part, int n_parts, cudaStream_t st,
                               const int64_t* offsets_host = nullptr);
int64_t shard_words(const batmap_collection* h, int p, int n_parts);
void shard_cols(const batmap_collection* h, size_t a, int p, int n_parts, int64_t* c0, int64_t* c1);
batmap_status emit_sorted_keys(uint64_t* keys, uint32_t* vals, int64_t K, int64_t cap, batmap_triple* out,
                               cudaStream_t st);
batmap_status merge_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items, const int32_t* items,
                                  int64_t n_sel, uint32_t threshold, batmap_triple* out, int64_t capacity,
                                  int64_t* n_out, double* kernel_ms, int64_t* merge_steps, cudaStream_t st);
batmap_status shard_copy(batmap_collection* h, int p, int n_parts, uint32_t* packed, bool to_arena, cudaStream_t st);
batmap_status shard_import(batmap_collection* h, const int64_t* offsets, const int32_t* tids,
                           const uint32_t* words_all, int64_t stride_words, const uint64_t* fails_all,
                           const int64_t* n_fails, int64_t stride_fails, cudaStream_t st);
// intersect.cu
struct TileList {
    std::vector<int4> tiles;  // (a, b, ti, tj)
    int64_t work = 0;
};
void plan_tiles(const std::vector<ClassInfo>& cls, int tile_m, int part, int n_parts, TileList* out);
batmap_status run_intersect(batmap_collection* h, const Selection& sel, uint32_t threshold,
                            int part, int n_parts, uint32_t flags, cudaStream_t st,
                            int64_t* n_cand);
batmap_status swar_device(const uint32_t* x, const uint32_t* y, int64_t n, uint32_t* out,
                          cudaStream_t st);
batmap_status prepare_full_k2(batmap_collection* h, int part, int n_parts, cudaStream_t st,
                              K2Prepared* host_plan = nullptr);
bool full_k2_plannable(const batmap_collection* h);
K2Prepared* new_k2_host_plan(const std::vector<ClassInfo>& classes, int num_sms, int part, int n_parts);
void destroy_k2(K2Prepared* kp, cudaStream_t st);
// finalize.cu
batmap_status run_finalize(batmap_collection* h, const Selection& sel, int64_t n_cand,
                           uint32_t threshold, uint32_t flags, cudaStream_t st, int64_t* n_res);
batmap_status gather_selection(batmap_collection* h, const int32_t* items_d, int64_t n_sel,
                               cudaStream_t st, Selection* sel);
batmap_status gather_selection_host(batmap_collection* h, const std::vector<int32_t>& items, cudaStream_t st,
                                    Selection* sel);
batmap_status sort_triples(batmap_triple* t, int64_t n, cudaStream_t st);
// ingest.cu
batmap_status fimi_parse(const uint8_t* text, int64_t n, cudaStream_t st, batmap_fimi* h, int64_t* bad_line);
batmap_status fimi_filter(batmap_fimi* h, uint32_t min_support, cudaStream_t st);
batmap_status frequent_items(const int64_t* off, int64_t n_items, uint32_t min_support, int32_t* items_out,
                             int64_t* n_out, cudaStream_t st);
batmap_status select_csr(const int64_t* off, const int32_t* tids, const int32_t* items, int64_t n_sel,
                         int64_t* offsets_out, int32_t* tids_out, int64_t tids_capacity, int64_t* nnz_out,
                         cudaStream_t st);
// dense.cu
batmap_status dense_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items, int64_t m,
                                  const int32_t* items, int64_t n_sel, uint32_t threshold, batmap_triple* out,
                                  int64_t capacity, int64_t* n_out, double* gemm_ms, cudaStream_t st);
}  // namespace bm
