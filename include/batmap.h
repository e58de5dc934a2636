/*
 * batmap.h -- C ABI of the B200-native BatMap all-pairs support counting library.
 *
 * The hot path of Amossen & Pagh, "A New Data Layout For Set Intersection on GPUs"
 * (arXiv 1102.1003; cited as P:<line> of /root/reference/PAPER.md):
 *
 *   vertical tidlists S_i
 *     --batmap_build-->          one BatMap per item: 2-of-3 cuckoo placement,
 *                                superblock layout, 8-bit entries with the
 *                                indicator bit as MSB, ⊥ = 0x7F
 *     --batmap_pair_supports-->  every selected pair intersected word by word with the
 *                                wrap-around SWAR compare-and-count (P:218-234, P:273-274,
 *                                P:423-431), failed insertions corrected, and
 *                                the pairs with support >= threshold emitted
 *
 * Conventions
 *   - Plain C types only.  Pointers are marked [device] (CUDA global memory) or [host].
 *   - Item ids are the caller's ids 0..n_items-1 (the row index of the input CSR);
 *     transaction ids are 0-based, 0 <= tid < n_transactions (reading #2).
 *   - Every call is stream-ordered on `stream` (a cudaStream_t; NULL = legacy default
 *     stream).  Calls that return a count (build, pair_supports) synchronise `stream`
 *     once to read it; all other device work stays asynchronous.
 *   - No C++ exception crosses the ABI.  On a non-OK status, batmap_last_error()
 *     returns a thread-local message.  A handle may be used by one thread at a time.
 *   - Out-of-memory is reported as BATMAP_E_NOMEM, CUDA runtime failures as
 *     BATMAP_E_CUDA.  After BATMAP_E_CUDA the handle must only be destroyed.
 */
#ifndef BATMAP_H_
#define BATMAP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BATMAP_OK = 0,
    BATMAP_E_INVALID = -1,   /* bad argument or input (see each function)            */
    BATMAP_E_NOMEM = -2,     /* device or host allocation failed                     */
    BATMAP_E_CUDA = -3,      /* CUDA runtime error; details in batmap_last_error()   */
    BATMAP_E_CAPACITY = -4,  /* output buffer too small; *n_out holds the size needed */
    BATMAP_E_OVERFLOW = -5   /* n_transactions >= 2^31, n_items >= 2^31, size overflow */
} batmap_status;

typedef struct CUstream_st* batmap_stream_t;   /* == cudaStream_t */
typedef struct batmap_collection* batmap_handle; /* library-owned; free with batmap_destroy */

/*
 * Environment switches (diagnostics and test hooks; read per call; every setting is exact, only the
 * speed differs):
 *   BATMAP_K1_BYTE=0|all      byte-table K1 tier never / for every class (default: measured policy)
 *   BATMAP_K1_SMALL, BATMAP_K1_SPREAD, BATMAP_K1_SIDE, BATMAP_K1_IPC   other K1 tier policies
 *   BATMAP_K1_STAGE=0|4       staged K1 pack off / byte tier also at 4 items per CTA (default: 1-2)
 *   BATMAP_K2_TN=64|128       K2 tile width (default: the planner's cost model)
 *   BATMAP_K2_PROMOTE=0, BATMAP_K2_VIRTUAL=0, BATMAP_K2_SPLIT=0        planner features off
 *   BATMAP_K2_SPLITF=f        split-K granularity (default 4); BATMAP_K2_ACCTAIL=0: no finer tail cut
 *   BATMAP_K2_GROUP=g         tile rows per band of large rectangles (default: ~32 MB bands)
 *   BATMAP_K2_BALANCE=0       K2's balanced mode for ragged / diagonal tiles off
 *   BATMAP_K3_GROUPED=0       the one-warp-per-candidate triple kernel instead of the grouped one
 *   BATMAP_AB_CAP=n           force the A_b re-run path;  BATMAP_TRACE=1|2: host phase / plan-upload timestamps (stderr)
 */

/* Build flags */
#define BATMAP_CHECK_INPUT 0x1u   /* validate on device: every tidlist strictly increasing, 0 <= tid < m */
#define BATMAP_BUILD_SERIAL 0x2u  /* one thread runs each item's INSERTs in ascending tid order:
                                     deterministic bytes, slower.  Default: the INSERTs of an item run
                                     concurrently (atomic swaps); layout timing-dependent, supports identical */

/* pair_supports flags (batmap_pair_supports_ex) */
#define BATMAP_PAIRS_RAW 0x1u      /* test hook: emit the raw BatMap counts (no failure corrections) */
#define BATMAP_PAIRS_SIMPLE 0x2u   /* test hook: use the one-thread-per-pair kernel (cross-check)    */
#define BATMAP_PAIRS_FREQUENT 0x4u /* intersect only items with |S_i| >= threshold (no pair with an
                                      infrequent item reaches the threshold); same output, less work.
                                      Ignored for threshold 0 and with BATMAP_PAIRS_RAW */

/*
 * Build options.  Zero-initialised = defaults.
 *   seed      seeds the three permutations π_1..π_3 (reading #3).
 *   r_min     floor on every table range r_i; power of two >= 4.  0 => 128.  With r_min
 *             >= 128 every BatMap is a multiple of 32 words, which the tiled intersection
 *             kernel requires; smaller values fall back to the simple kernel.
 *   max_loop  MaxLoop rounds of INSERT.  0 => 16 + ceil(3 log2 r_i).
 *   flags     BATMAP_CHECK_INPUT | BATMAP_BUILD_SERIAL.
 *   pi_table  [device] test hook: 3 x U uint32 table replacing the mixer (row t-1 = π_t),
 *             each row a permutation of [0, U), U = 127 * 2^s.  NULL => seeded mixer.
 *             Read during batmap_build only.
 */
typedef struct {
    uint64_t seed;
    uint32_t r_min;
    uint32_t max_loop;
    uint32_t flags;
    uint32_t reserved;
    const uint32_t* pi_table;
} batmap_build_opts;

/* One output record: i < j in caller ids; support = |S_i ∩ S_j|. */
typedef struct {
    uint32_t i, j, support;
} batmap_triple;

typedef struct {
    int32_t s_shift;      /* s: entries store π_t(x) >> s                 */
    int32_t n_classes;    /* distinct table ranges r among the items             */
    int64_t U;            /* permutation domain 127 * 2^s                        */
    int64_t r0;           /* min_i r_i (|B_0| = 3 r0)                     */
    int64_t n_items;
    int64_t n_transactions;
    int64_t arena_bytes;  /* sum_i 3 r_i (the BatMaps, without padding)          */
    int64_t n_failures;   /* |F|: (item, tid) insertions that failed */
    int64_t n_failed_tids;/* distinct transactions b with F_b non-empty          */
} batmap_info_t;

/*
 * batmap_build -- construct the BatMap of every item.
 *   offsets   [device] int64[n_items+1], offsets[0] = 0, non-decreasing: item i's tidlist
 *             is tids[offsets[i] .. offsets[i+1]).
 *   tids      [device] int32[offsets[n_items]]: each tidlist strictly increasing,
 *             0 <= tid < n_transactions (validated only with BATMAP_CHECK_INPUT).  May be NULL
 *             when offsets[n_items] == 0 (every tidlist empty; a zero-length array); the same
 *             holds for the tids of batmap3_build, batmap_dense_pair_supports and
 *             batmap_merge_pair_supports.
 *   n_items, n_transactions   n and m; 1 <= m < 2^31, 0 <= n < 2^31.
 *   opts      [host] may be NULL (defaults).
 *   out       [host] receives the handle.
 * The handle owns the BatMaps (HBM), the failure list F, per-item failure counts and
 * the item lists A_b of failed transactions.  The input CSR is read during the
 * call only and may be freed once `stream` has completed this call's work.
 * Errors: E_INVALID (null pointer, bad offsets, r_min not a power of two >= 4, invalid
 * tidlists in checked mode), E_OVERFLOW, E_NOMEM, E_CUDA.
 */
batmap_status batmap_build(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                           int64_t n_transactions, const batmap_build_opts* opts,
                           batmap_stream_t stream, batmap_handle* out);

/*
 * batmap_pair_supports -- all pairs {i, j} of the selected items with
 * |S_i ∩ S_j| >= threshold, as triples (i < j, caller ids) sorted by (i, j).
 *   items     [device] int32[n_sel] distinct caller ids, or NULL => all items.
 *   threshold emit iff support >= threshold (inclusive); 0 => every pair,
 *             including zero supports.
 *   out       [device] caller-owned, capacity records.
 *   n_out     [host] number of records; also set on E_CAPACITY (the size needed).
 * On E_CAPACITY the computed result is kept in the handle: an immediately following
 * call with the same arguments (same items pointer and contents) and enough capacity
 * returns it without recomputation.
 * Errors: E_INVALID (null handle/out/n_out, duplicate or out-of-range items),
 * E_CAPACITY, E_NOMEM, E_CUDA.
 */
batmap_status batmap_pair_supports(batmap_handle h, const int32_t* items, int64_t n_sel,
                                   uint32_t threshold, batmap_triple* out, int64_t capacity,
                                   int64_t* n_out, batmap_stream_t stream);

/*
 * batmap_pair_supports_part -- the share of rank `part` (0 <= part < n_parts) of the
 * pairs of batmap_pair_supports: the work tiles of the pair triangle are
 * ordered by cost and dealt round-robin to the parts, so the union over parts is
 * exactly the full result and the parts are disjoint.  Output sorted by (i, j).
 */
batmap_status batmap_pair_supports_part(batmap_handle h, const int32_t* items, int64_t n_sel,
                                        uint32_t threshold, int32_t part, int32_t n_parts,
                                        batmap_triple* out, int64_t capacity, int64_t* n_out,
                                        batmap_stream_t stream);

/*
 * Sharded build for multi-GPU runs (the paper is single-GPU).
 * Every BatMap depends on its own tidlist only, so part `part` of `n_parts`
 * builds the BatMaps of a contiguous share of each width class (columns
 * [n_c*part/n_parts, n_c*(part+1)/n_parts) of class c, n_c its item count) and records
 * the failures of those items; the parts then exchange their shares (an all_gather of
 * batmap_shard_export's buffers, done by the caller, e.g. torch.distributed over NCCL)
 * and batmap_shard_import completes the handle, after which it is identical in use to a
 * batmap_build handle.  Until then batmap_pair_supports* return E_INVALID.
 *
 * batmap_build_shard -- arguments as batmap_build plus 0 <= part < n_parts.  The CSR must
 *   be the full collection on every part (the same arrays on every rank).
 * batmap_shard_sizes -- words (uint32) of part p's share of the BatMaps (any p: the layout
 *   is computed identically on every rank) and, for p == this part, its number of
 *   failure records (else -1).
 * batmap_shard_export -- [device] words_out <- this part's share, as a packed
 *   [class][word][column] array; [device] fails_out <- its failure records (opaque uint64).
 *   E_CAPACITY if a buffer is smaller than batmap_shard_sizes reports.
 * batmap_shard_import -- [device] words_all = n_parts blocks of stride_words words, block p
 *   = part p's export; [device] fails_all = n_parts blocks of stride_fails records, block p
 *   holding n_fails[p] ([host] int64[n_parts]) records; offsets/tids [device] the same CSR
 *   as the build (A_b of the failed transactions is rebuilt from it).  Copies the
 *   other parts' BatMaps into place, merges F and derives f_i, Fail(i) and A_b exactly as a
 *   whole build does; synchronises `stream`.  E_INVALID on a handle that is not a pending
 *   shard, NULL buffers, or counts that do not fit the strides or disagree with this part.
 */
batmap_status batmap_build_shard(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                                 int64_t n_transactions, const batmap_build_opts* opts,
                                 int32_t part, int32_t n_parts, batmap_stream_t stream,
                                 batmap_handle* out);
batmap_status batmap_shard_sizes(batmap_handle h, int32_t part, int64_t* words, int64_t* n_fail);
batmap_status batmap_shard_export(batmap_handle h, uint32_t* words_out, int64_t words_capacity,
                                  uint64_t* fails_out, int64_t fails_capacity,
                                  batmap_stream_t stream);
batmap_status batmap_shard_import(batmap_handle h, const int64_t* offsets, const int32_t* tids,
                                  const uint32_t* words_all, int64_t stride_words,
                                  const uint64_t* fails_all, const int64_t* n_fails,
                                  int64_t stride_fails, batmap_stream_t stream);

/* General form: flags = BATMAP_PAIRS_FREQUENT, and the test hooks BATMAP_PAIRS_RAW | BATMAP_PAIRS_SIMPLE. */
batmap_status batmap_pair_supports_ex(batmap_handle h, const int32_t* items, int64_t n_sel,
                                      uint32_t threshold, int32_t part, int32_t n_parts,
                                      uint32_t flags, batmap_triple* out, int64_t capacity,
                                      int64_t* n_out, batmap_stream_t stream);

/* batmap_info -- parameters of a built collection.  info [host].  E_INVALID on NULL. */
batmap_status batmap_info(batmap_handle h, batmap_info_t* info);

/* batmap_destroy -- release everything the handle owns (stream-ordered).  NULL is a no-op. */
void batmap_destroy(batmap_handle h);

/* batmap_last_error -- thread-local message for the last non-OK status ("" if none). */
const char* batmap_last_error(void);

/* batmap_version -- library version string. */
const char* batmap_version(void);

/*
 * batmap_mine_host -- end-to-end call on HOST buffers: copies the CSR to the device,
 * builds, computes the pairs, copies the triples back and frees the device state.
 *   offsets, tids, items [host] as in batmap_build / batmap_pair_supports (items may be NULL).
 *   out [host] capacity records; n_out [host] (set also on E_CAPACITY).
 */
batmap_status batmap_mine_host(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                               int64_t n_transactions, const batmap_build_opts* opts,
                               const int32_t* items, int64_t n_sel, uint32_t threshold,
                               batmap_triple* out, int64_t capacity, int64_t* n_out,
                               batmap_stream_t stream);

/*
 * batmap_stats -- measurements of the last batmap_build and batmap_pair_supports* calls on
 * this handle.  Device times come from CUDA events recorded on the launching stream around
 * each phase.  word_compares is the algorithmic work of the intersection:
 * the sum over the selected pairs of this part of max(W_i, W_j), W = 3r/4 words;
 * tile_compares is what the kernel executed (tile padding and diagonal tiles included).
 * launches_* count the kernels this library launched (its own and its CUB sorts/scans).
 */
typedef struct {
    double build_ms;        /* batmap_build, device time of all its work                 */
    double k1_insert_ms;    /* ★K1 cuckoo insertion kernel                                */
    double k1_encode_ms;    /* ★K1 encode kernel(s)                                       */
    double pairs_ms;        /* batmap_pair_supports*, device time of all its work         */
    double k2_ms;           /* ★K2 intersection kernel (one launch)                       */
    double k3_ms;           /* ★K3 correction + sort                                      */
    int64_t word_compares;
    int64_t tile_compares;
    int64_t n_candidates;   /* K2 epilogue candidates (c + f_i + f_j >= threshold)        */
    int64_t n_results;
    int32_t k2_kind;        /* 1 = tiled TMA kernel, 2 = one-thread-per-pair kernel        */
    int32_t k2_grid;        /* CTAs launched for K2                                        */
    int64_t launches_build;
    int64_t launches_pairs;
    double build_pre_ms;    /* batmap_build up to the insertion kernel (offsets read-back, host
                               planning, uploads, padding fill) as seen on the stream          */
    double build_post_ms;   /* batmap_build after the encode (failure list F, Fail(i), A_b)     */
    int32_t k2_tile_cols;   /* tiled K2: tile width in items (128, or 64 for small/ragged plans)  */
    int32_t reserved;
    int64_t n_selected;     /* items intersected by the last pair_supports (after BATMAP_PAIRS_FREQUENT) */
} batmap_stats_t;

batmap_status batmap_stats(batmap_handle h, batmap_stats_t* out);

/*
 * batmap_sort_triples -- sort triples in place by (i, j) on the device (used to merge the
 * parts gathered from several ranks).  triples [device] n records.
 */
batmap_status batmap_sort_triples(batmap_triple* triples, int64_t n, batmap_stream_t stream);

/*
 * batmap_dense_pair_supports -- NEXT-1 comparison path, NOT the BatMap method: the same triples
 * computed from dense bitmaps, i.e. the integer matrix product X^T X of the
 * m x n 0/1 incidence matrix on the tensor cores (cuBLASLt int8 GEMM, int32 accumulation, upper
 * triangle in row blocks), thresholded and sorted by (i, j).  No handle, no failures.
 *   offsets, tids [device] CSR as in batmap_build (valid tidlists assumed);
 *   items [device] distinct caller ids or NULL (all); out [device] capacity records;
 *   n_out [host] (set also on E_CAPACITY); gemm_ms [host] or NULL: device time of GEMM+threshold.
 * Memory: n_sel x m bytes for X (E_NOMEM above 48 GB) plus one 512 MB block of X^T X.
 * cuBLASLt is loaded on first use; E_CUDA if it cannot be loaded.
 */
batmap_status batmap_dense_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                                         int64_t n_transactions, const int32_t* items, int64_t n_sel,
                                         uint32_t threshold, batmap_triple* out, int64_t capacity,
                                         int64_t* n_out, double* gemm_ms, batmap_stream_t stream);

/*
 * batmap_merge_pair_supports -- NEXT-2 comparison path, NOT the BatMap method: the same triples
 * by sorted-list merging (a + b steps per pair of lengths a, b), the
 * intersection the paper compares BatMaps with.  Arguments as batmap_dense_pair_supports;
 * kernel_ms [host] or NULL: device time of the merge kernel; merge_steps [host] or NULL: the
 * algorithmic step count sum over pairs of (a + b).  Tidlists must be strictly increasing.
 */
batmap_status batmap_merge_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                                         int64_t n_transactions, const int32_t* items, int64_t n_sel,
                                         uint32_t threshold, batmap_triple* out, int64_t capacity,
                                         int64_t* n_out, double* kernel_ms, int64_t* merge_steps,
                                         batmap_stream_t stream);

/* ---------------------------------------------------------------- inspection / test hooks */

/*
 * Determinism of the exported bytes: the default build inserts the elements of an item
 * concurrently (reading #9b in DESIGN.md), so the entry bytes and the failure set F may differ
 * from build to build of the same input; the pair supports never do (every layout is exact
 * after the corrections).  Builds with BATMAP_BUILD_SERIAL follow the paper's
 * sequential INSERT in ascending tid order and are byte-reproducible for identical
 * (tidlists, seed, r_min, max_loop).
 *
 * batmap_export_entries -- the 3 r_i entry bytes of item `item` in entry order
 * e = 0 .. 3 r_i - 1 (superblock layout P:378-379, 4 entries per little-endian word).
 *   out [host] capacity bytes; r_out [host] receives r_i.  E_CAPACITY if capacity < 3 r_i.
 */
batmap_status batmap_export_entries(batmap_handle h, int32_t item, uint8_t* out,
                                    int64_t capacity, int64_t* r_out);

/*
 * batmap_export_failures -- F as (item, tid) pairs sorted by (item, tid).
 *   items, tids [host] capacity entries each; n_out [host].  E_CAPACITY if too small.
 */
batmap_status batmap_export_failures(batmap_handle h, int32_t* items, int32_t* tids,
                                     int64_t capacity, int64_t* n_out);

/*
 * batmap_swar_device -- runs the device compare routines on word pairs:
 *   out[k]     = matches of (x[k], y[k]) by the intersection kernel's 4-instruction form,
 *   out[n + k] = matches by the paper's literal formula.
 *   x, y [device] uint32[n]; out [device] uint32[2n].
 */
batmap_status batmap_swar_device(const uint32_t* x, const uint32_t* y, int64_t n, uint32_t* out,
                                 batmap_stream_t stream);

/*
 * batmap_plan_work -- host-only view of the intersection planner (no device needed).  For width
 * classes a = 0..n_classes-1 with class_n[a] items of class_w[a] words (class_w ascending, each a
 * multiple of 16), lists the work items of `part` of `n_parts` in execution order.  A work item is
 * the 128 x tile_cols tile (ti, tj) (see batmap_plan_tile) of the class rectangle (a, b) of PLANNED classes (see
 * batmap_plan_groups; equal to the input classes when nothing is promoted), a <= b (tj >= ti when a == b), over
 * k-chunks [k0, k1) of 16 words; R > 1 marks a virtualised rectangle (each class-b BatMap viewed as
 * R columns of class_w[a] words); acc = 1 marks rectangles whose partial counts are summed in
 * global counters (virtualised or split along k).
 *   grid_cap  resident CTAs assumed for the split-K target (0 => 2 x 148, or 4 x 148 for 64-wide tiles).
 *   items     [host] 8 * capacity int32: (a, b, ti, tj, k0, k1, R, acc) per item.
 *   n_items, word_compares, tile_compares [host]: count; sum over this part's pairs of
 *             max(W_i, W_j); words x 128 x tile_cols summed over its items.
 */
batmap_status batmap_plan_work(int32_t n_classes, const int64_t* class_n, const int64_t* class_w,
                               int32_t part, int32_t n_parts, int32_t grid_cap, int32_t* items,
                               int64_t capacity, int64_t* n_items, int64_t* word_compares,
                               int64_t* tile_compares);

/* ------------------------------------------------------------------------------------------
 * NEXT-3: FIMI-repository text -> vertical tidlists, and the frequent-item filter.
 *
 * The paper's real-data experiment reads a file "taken from the Frequent Itemset Mining Dataset
 * Repository" -- one transaction per line, whitespace-separated item labels -- and
 * the method starts from the vertical layout.  It also assumes the data "preprocessed
 * ... to remove items with support below the threshold".  Semantics (
 * readings #21-#25 in DESIGN.md):
 *   - transaction id = 0-based line index; the text after the last '
' is a transaction iff it
 *     is non-empty; blank lines are empty transactions;
 *   - a label is a run of decimal digits, 0 <= label <= 2^32 - 1; separators are ' ', '	', '
';
 *     any other byte, or a longer number, is an error;
 *   - duplicate labels within a line collapse (set semantics);
 *   - items are re-densified: dense id k is the k-th smallest label present; labels[k] maps back.
 * ------------------------------------------------------------------------------------------ */
typedef struct batmap_fimi* batmap_fimi_handle; /* library-owned; free with batmap_fimi_destroy */

/*
 * batmap_fimi_parse -- parse FIMI text into a library-owned vertical database.
 *   text      [device] n_bytes bytes (any alignment; 16-byte aligned is read with 128-bit loads).
 *             Read-only; may be freed once the call returns.
 *   out       [host] receives the handle (NULL on error).
 *   bad_line  [host] 1-based line of the first offending byte / oversized label on E_INVALID,
 *             else -1.
 * Synchronises `stream` (three times: token count, errors, item count).
 * Errors: E_INVALID (null pointer, n_bytes < 0, malformed text), E_OVERFLOW (>= 2^31
 * transactions), E_NOMEM, E_CUDA.
 */
batmap_status batmap_fimi_parse(const uint8_t* text, int64_t n_bytes, batmap_stream_t stream,
                                batmap_fimi_handle* out, int64_t* bad_line);

/* Sizes of the parsed (and possibly filtered) database: items, (item, tid) pairs, transactions. */
batmap_status batmap_fimi_info(batmap_fimi_handle h, int64_t* n_items, int64_t* nnz,
                               int64_t* n_transactions);

/*
 * batmap_fimi_filter -- keep only the items with support |S_i| >= min_support, in
 * ascending dense-id (= label) order; labels follow; n_transactions unchanged.  min_support 0
 * keeps everything.  Synchronises `stream`.
 */
batmap_status batmap_fimi_filter(batmap_fimi_handle h, uint32_t min_support, batmap_stream_t stream);

/*
 * batmap_fimi_export -- copy the database into caller-owned device buffers (any may be NULL):
 *   offsets [device] n_items + 1 int64; tids [device] nnz int32 (each list strictly increasing);
 *   labels [device] n_items uint32.  The CSR is exactly what batmap_build takes.  Asynchronous.
 */
batmap_status batmap_fimi_export(batmap_fimi_handle h, int64_t* offsets, int32_t* tids, uint32_t* labels,
                                 batmap_stream_t stream);

void batmap_fimi_destroy(batmap_fimi_handle h);

/*
 * batmap_frequent_items -- the frequent-item pre-filter on any vertical CSR: the ids
 * i with offsets[i+1] - offsets[i] >= min_support, ascending, written to items_out (a selection
 * for batmap_pair_supports: a pair with support >= s has both items frequent).
 *   offsets    [device] n_items + 1;  items_out [device] capacity n_items;  n_out [host].
 * Synchronises `stream`.  Errors: E_INVALID (null pointers, n_items < 0), E_OVERFLOW (n_items >= 2^31).
 */
batmap_status batmap_frequent_items(const int64_t* offsets, int64_t n_items, uint32_t min_support,
                                    int32_t* items_out, int64_t* n_out, batmap_stream_t stream);

/*
 * batmap_select_csr -- the vertical database restricted to the items `items` (in that order; e.g.
 * the output of batmap_frequent_items): offsets_out [device, n_sel + 1] is always written;
 * tids_out [device, tids_capacity] receives the selected tidlists back to back.  *nnz_out [host] =
 * their total length; if it exceeds tids_capacity the call returns E_CAPACITY after writing
 * offsets_out (two-call protocol).  `items` are ids in [0, n_items) (not validated; duplicates are
 * copied twice).  Synchronises `stream` once.  Errors: E_INVALID, E_CAPACITY, E_NOMEM, E_CUDA.
 */
batmap_status batmap_select_csr(const int64_t* offsets, const int32_t* tids, int64_t n_items, const int32_t* items,
                                int64_t n_sel, int64_t* offsets_out, int32_t* tids_out, int64_t tids_capacity,
                                int64_t* nnz_out, batmap_stream_t stream);

/*
 * batmap_plan_groups -- host-only view of the planner's class promotion (no device needed).  The
 * planner may merge a run of adjacent width classes (typically small, narrow ones whose own
 * 128 x 128 tiles would be mostly padding) into ONE planned class of the widest member's width W:
 * each narrower BatMap is replicated along k, B'[w] = B[w mod W_i] (valid because every width is
 * 3r/4 with r a power of two, so W_i | W).  A pair of planned widths then compares K words, which
 * is K / max(W_i, W_j) times the wrap-around count of P:218-219; the epilogue divides
 * exactly.  Same input conventions as batmap_plan_work.  Set the environment variable
 * BATMAP_K2_PROMOTE=0 to disable promotion (both here and in batmap_pair_supports*).
 *   group_of  [host] n_classes int32: planned class of each input class (non-decreasing; the
 *             `a`, `b` of batmap_plan_work's items index these planned classes).
 * Errors: E_INVALID on bad arguments.
 */
batmap_status batmap_plan_groups(int32_t n_classes, const int64_t* class_n, const int64_t* class_w,
                                 int32_t* group_of);

/*
 * batmap_plan_tile -- host-only view of the planner's tile shape (no device needed): tile_rows =
 * 128 items; tile_cols = 128, or 64 when the cost model finds that 128 x 64 tiles execute > 10 %
 * fewer compares (small or ragged width classes; 4 CTAs of 4 warps per SM instead of 2 of 8).
 * BATMAP_K2_TN=64|128 overrides.  The `tj` of batmap_plan_work's items counts tile_cols-wide
 * column tiles.  Same input conventions as batmap_plan_work.  Errors: E_INVALID.
 */
batmap_status batmap_plan_tile(int32_t n_classes, const int64_t* class_n, const int64_t* class_w,
                               int32_t* tile_rows, int32_t* tile_cols);

/* ------------------------------------------------------------------------------------------
 * NEXT-4: supports of item TRIPLES with 3-of-4 BatMaps.
 *
 * The paper leaves itemsets of more than two items open and sketches "a
 * generalization of batmaps that store items in d out of d+1 places", which "would ensure that
 * itemsets of size up to d would have at least one position witnessing their intersection".
 * These entry points build that structure for d = 3 and count triples with it.  The counting
 * rule that makes every common element count exactly once is not in the paper: readings
 * #26-#32 of DESIGN.md fix it (oracle/batmap3_ref.py follows them step by step):
 *   - four tables, permutations π_1..π_4 (the mixer of reading #3 with keys for t = 0..3);
 *   - 6-bit codes π_t(x) >> s3, s3 = min{s : 63 * 2^s >= m}, ⊥ = code 63; table ranges
 *     r_i = max(2^ceil(log2 2|S_i|), 2^s3, r_min); superblocks of 4 r_0, 4 r_i bytes per item;
 *   - INSERT over A_1..A_4 cyclically, three times per element; failed insertions are deleted
 *     and corrected exactly, as for pairs (P:469-474 with set semantics per triple);
 *   - entry byte = code | B1 << 6 | B2 << 7 encoding which table leaves the element out, and a
 *     triple is counted at the lowest table all three BatMaps store the element in.
 * Output = the definition supp(i,j,k) = |S_i ∩ S_j ∩ S_k|, bit-exact.
 * ------------------------------------------------------------------------------------------ */
typedef struct batmap3_collection* batmap3_handle; /* library-owned; free with batmap3_destroy */

/* One triple record: i < j < k caller ids; support = |S_i ∩ S_j ∩ S_k|. */
typedef struct {
    uint32_t i, j, k, support;
} batmap_quad;

typedef struct {
    int32_t s_shift;       /* s3: entries store π_t(x) >> s3                       */
    int32_t reserved;
    int64_t r0;            /* min_i r_i (superblocks of 4 r0 entries)             */
    int64_t n_items;
    int64_t n_transactions;
    int64_t arena_bytes;   /* sum_i 4 r_i                                         */
    int64_t n_failures;    /* |F| of the 3-of-4 build                             */
    int64_t n_failed_tids;
    double build_ms;       /* CUDA-event time of batmap3_build                    */
    double triples_ms;     /* CUDA-event time of the last batmap3_triple_supports */
} batmap3_info_t;

/*
 * batmap3_build -- the 3-of-4 BatMap of every item.  Same input contract as batmap_build
 * (offsets/tids [device] CSR, n_items < 2^21, 1 <= n_transactions < 2^31; opts: seed, r_min,
 * max_loop (rounds of four swaps), flags BATMAP_CHECK_INPUT | BATMAP_BUILD_SERIAL, pi_table =
 * [device] 4 x U3 test table, U3 = 63 * 2^s3).  The handle owns the BatMaps (item-major,
 * 4 r_i bytes each), F, f_i and A_b of failed transactions; the CSR is read during the call
 * only (the call synchronises `stream` before returning).
 * Errors: E_INVALID, E_OVERFLOW, E_NOMEM, E_CAPACITY (failure buffer), E_CUDA.
 */
batmap_status batmap3_build(const int64_t* offsets, const int32_t* tids, int64_t n_items,
                            int64_t n_transactions, const batmap_build_opts* opts,
                            batmap_stream_t stream, batmap3_handle* out);

/*
 * batmap3_triple_supports -- supports of candidate triples, thresholded.
 *   triples   [device] int32 [n_triples][3]: caller ids i < j < k (not checked).
 *   threshold emit iff support >= threshold (0 => every candidate).
 *   out       [device] batmap_quad[capacity], sorted by (i, j, k); n_out [host] receives the
 *             count (set also on E_CAPACITY).
 * One warp per candidate counts over the words of its widest BatMap (the others wrap, reading
 * #18) with reading #30's rule; candidates with count + f_i + f_j + f_k >= threshold get the
 * exact correction of reading #31.
 */
batmap_status batmap3_triple_supports(batmap3_handle h, const int32_t* triples, int64_t n_triples,
                                      uint32_t threshold, batmap_quad* out, int64_t capacity,
                                      int64_t* n_out, batmap_stream_t stream);

/*
 * batmap_candidate_triples -- Apriori join (reading #32): every i < j < k such that (i, j),
 * (i, k) and (j, k) all occur in `pairs`.
 *   pairs  [device] batmap_triple[n_pairs] sorted by (i, j) with i < j < n_items, as
 *          batmap_pair_supports returns them (the frequent pairs).
 *   out    [device] int32 [capacity][3], sorted by (i, j, k); n_out [host] (set also on
 *          E_CAPACITY).
 * Exact for frequent-triple mining: supp(i,j,k) <= the support of each of its pairs.
 */
batmap_status batmap_candidate_triples(const batmap_triple* pairs, int64_t n_pairs, int64_t n_items,
                                       int32_t* out, int64_t capacity, int64_t* n_out,
                                       batmap_stream_t stream);

batmap_status batmap3_info(batmap3_handle h, batmap3_info_t* info);
/* batmap3_export_entries -- item's 4 r_i entry bytes [host] (E_CAPACITY if capacity < 4 r_i). */
batmap_status batmap3_export_entries(batmap3_handle h, int32_t item, uint8_t* out, int64_t capacity,
                                     int64_t* r_out);
/* batmap3_export_failures -- F as (item, tid) [host] sorted by (item, tid). */
batmap_status batmap3_export_failures(batmap3_handle h, int32_t* items, int32_t* tids,
                                      int64_t capacity, int64_t* n_out);
void batmap3_destroy(batmap3_handle h);

#ifdef __cplusplus
}
#endif
#endif /* BATMAP_H_ */
