// plan.h -- host-side work planner of ★K2 (shared by intersect.cu and the C ABI's plan hook).
#pragma once

#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace bm {

constexpr int kTile = 128;   // tile rows (items); the tile width (columns) is Plan::tn, 128 or 64
constexpr int kChunk = 16;   // words per k-chunk (the TMA box height)
constexpr int kDealGrid = 2 * 148;  // reference grid (B200: 2 K2 CTAs x 148 SMs) for rank-agreed plan decisions

// A rectangle of the pair triangle: the rows are the items of class a (period W_a), the
// columns those of class b.  A "virtualised" rectangle (R > 1) views each class-b BatMap of
// W_b = R W_a words as R virtual columns of W_a words each (column v = j R + rep holds words
// [rep W_a, (rep+1) W_a) of item j), so skinny rectangles (few wide items) tile densely:
// c_ij = sum_rep c(i, (j, rep))  (the wrap-around of P:273-274 unrolled).
struct Rect {
    int32_t cls_a, cls_b;         // selection classes
    int32_t map_a, map_b;         // tensor-map indices (map_b = virtual copy when R > 1)
    int32_t W_a, W;               // row period; K length of the rectangle (words)
    int32_t n_rows, n_cols;       // n_cols counts virtual columns when R > 1
    int32_t row_first, col_first; // selection index of the first row / first real column item
    int32_t diag, R;              // diag: a == b (pairs i < j only)
    int32_t acc, n_cols_real;     // acc: partial counts accumulate into cnt[] (virtual or split-K)
    int64_t cnt_off;              // offset of this rectangle's n_rows x n_cols_real counters
    int32_t promo;                // rows or columns include promoted (replicated) items
    int32_t lgK;                  // log2 of the rectangle's real width in units of the smallest W
};

struct Work {   // one work item: tile (ti, tj) of a rectangle over k-chunks [k0, k1)
    int32_t rect, ti, tj, k0, k1;
    int32_t tail;  // 0, or 1 + the slice of the tail buffer this piece of a cut tail tile writes
};

// Storage of work lists: large blocks (>= 1 MB) come from a process-wide pool and are kept, already
// faulted in, for the next plan (C4's 7.6 MB list: first-touch page faults cost 0.5-4 ms per
// build on the host); smaller ones from the heap.  Thread-safe.
void* plan_pool_alloc(size_t bytes);
void plan_pool_free(void* p);

template <class T>
struct PoolAlloc {
    using value_type = T;
    PoolAlloc() = default;
    template <class U>
    PoolAlloc(const PoolAlloc<U>&) {}
    T* allocate(size_t n) { return static_cast<T*>(plan_pool_alloc(n * sizeof(T))); }
    void deallocate(T* p, size_t) { plan_pool_free(p); }
    template <class U>
    bool operator==(const PoolAlloc<U>&) const { return true; }
    template <class U>
    bool operator!=(const PoolAlloc<U>&) const { return false; }
};
using WorkList = std::vector<Work, PoolAlloc<Work>>;

// K2's balanced mode (intersect.cu): in a ragged or diagonal tile the warps' fixed 32 x 16 blocks
// hold unequal numbers of valid pairs; dealing the valid blocks' k-steps evenly over the warps pays
// when the busiest warp would otherwise run at least 1/16 longer than the even share, and each warp's
// contiguous share then touches at most 4 blocks.  Evaluated identically on the host (which gives
// ordinary tiles that will run balanced a slice of the tail buffer) and in the kernel.
__host__ __device__ inline bool k2_block_valid(int n_rows, int n_cols, int diag, int ti, int tj, int tn, int rb,
                                               int cb) {
    const int r0 = ti * kTile + 32 * rb, c0 = tj * tn + 16 * cb;
    return r0 < n_rows && c0 < n_cols && !(diag && r0 >= c0 + 15);
}
__host__ __device__ inline bool k2_balance_pays(int n_rows, int n_cols, int diag, int ti, int tj, int tn) {
    const int nw = tn / 16, ncb = tn / 16;  // warps per CTA; 16-column groups per tile
    int B = 0, dmax = 0;
    for (int rb = 0; rb < 4; ++rb)
        for (int cb = 0; cb < ncb; ++cb) B += k2_block_valid(n_rows, n_cols, diag, ti, tj, tn, rb, cb);
    for (int w = 0; w < nw; ++w) {  // default: warp w owns row groups (w & 1) + {0, 2}, columns (w >> 1) + {0, ncb / 2}
        int c = 0;
        for (int t = 0; t < 4; ++t)
            c += k2_block_valid(n_rows, n_cols, diag, ti, tj, tn, (w & 1) + 2 * (t >> 1), (w >> 1) + (ncb / 2) * (t & 1));
        dmax = dmax > c ? dmax : c;
    }
    const int total = 16 * B, bmax = (total + nw - 1) / nw;
    if (B == 0 || bmax + bmax / 16 >= 16 * dmax) return false;  // a unit loads 2x the operands per compare
    for (int w = 0; w < nw; ++w) {
        const int lo = w * total / nw, hi = (w + 1) * total / nw;
        if (hi > lo && (hi - 1) / 16 - lo / 16 + 1 > 4) return false;
    }
    return true;
}

struct TailTile {  // a whole tile of an ordinary rectangle, cut into pieces at the end of the schedule
    int32_t rect, ti, tj, pad;
};

struct AccUnit {  // a tile row (rect, ti) of an accumulated rectangle owned by this part
    int32_t rect, ti;
};

struct VirtCopy {  // materialise class b's BatMaps as R virtual columns of period W_a
    int32_t cls_b, W_a, R, vpad;
    int64_t dst_word_off;  // into the virtual-copy scratch arena
};

// Promotion: a run of adjacent (narrow, small) width classes [cls_lo, cls_hi] is planned as ONE
// class of the widest member's width W.  Each narrower BatMap is replicated along k,
// B'[w] = B[w mod W_i] (W_i | W), into a word-major scratch block, so the members share tiles
// instead of each padding its own.  A pair then compares K = the rectangle's real width words,
// K / max(W_i, W_j) times the wrap-around count of P:273-274 (all widths are 3 r / 4 with r a
// power of two), and the epilogue divides exactly: c = c' >> (lgK - max(lw_i, lw_j)).
struct PromoCopy {
    int32_t cls_lo, cls_hi;  // original classes merged (ascending width)
    int32_t W, n, n_pad;     // promoted class: width, items, padded items
    int32_t pad;
    int64_t dst_word_off;    // into the promotion scratch arena
};

struct Plan {
    std::vector<ClassInfo> eff;   // the planned classes (original, or promoted groups)
    std::vector<int32_t> eff_of;  // original class -> planned class
    std::vector<PromoCopy> promo; // planned class -> copy, for promoted groups (eff[k].word_off is
                                  // then an offset into the promotion arena)
    std::vector<int32_t> eff_promo;  // planned class -> index into promo, or -1
    int64_t promo_words = 0;
    std::vector<Rect> rects;
    WorkList work;                // this part's work items, longest first
    std::vector<AccUnit> units;   // this part's tile rows of accumulated rectangles
    std::vector<VirtCopy> virt;
    std::vector<TailTile> tails;  // cut tail tiles; piece p of tail t writes slice t * tail_pieces + p
    int32_t tail_pieces = 0;
    int64_t virt_words = 0;
    int64_t cnt_entries = 0;
    int64_t word_compares = 0;    // algorithmic: sum over this part's pairs of max(W_i, W_j)
    int64_t tile_compares = 0;    // executed: sum over work items of 128 x tn x words
    int32_t tn = kTile;           // tile width: 128 x 128 tiles, or 128 x 64 for small / ragged plans
};

// grid_cap: CTAs the kernel keeps resident (the split-K target is ~4 work items per CTA).
// Rectangles, work items and units refer to the planned classes out->eff.
// tn: tile width (columns), 128 or 64.
void plan_work(const std::vector<ClassInfo>& cls, int part, int n_parts, int grid_cap, bool allow_virtual,
               bool allow_split, bool allow_promote, Plan* out, int tn = kTile);

// Estimated executed compares of the plan of `cls` with tile width tn (the planner's cost model,
// promotion and virtualisation included): used to choose tn.
int64_t plan_cost(const std::vector<ClassInfo>& cls, bool allow_virtual, bool allow_promote, int tn);

// 64 or 128 (see plan.cu); BATMAP_K2_TN overrides.
int choose_tn(const std::vector<ClassInfo>& cls, bool allow_virtual, bool allow_promote);

// log2 of W / W_min for a width that is W_min times a power of two (else -1)
int lg_ratio(int64_t W, int64_t W_min);

}  // namespace bm
