// intersect.cu -- ★K2: all-pairs BatMap intersection with the fused threshold epilogue.
//
// What is computed: for every selected pair (i, j) with
// W_i <= W_j words,   c_ij = sum_{w < W_j} SWAR(B_j[w], B_i[w mod W_i]),
// SWAR(x, y) = #byte lanes with equal 7 element bits and (b_x OR b_y).
//
// How (B200): the planner (plan.cu) cuts the pair triangle into width-class rectangles
// and 128 x 128 (or 128 x 64) tiles (symmetry cut p <= q); skinny rectangles are
// virtualised and long tiles split along k.  A persistent kernel, 2 CTAs x 8 warps per SM,
// claims work items longest-first from a global counter; thread 0 of each CTA streams
// [16 words x 128 items] boxes of both operands with TMA (cp.async.bulk.tensor, 3-stage mbarrier
// ring) -- the narrow operand's box coordinate is taken mod W_i, which realises the paper's
// wrap-around -- and every thread computes an 8 x 8 register micro-tile of pairs.  Per word pair
// the SWAR compare-and-count is 4 integer instructions (LOP3, IADD, LOP3, IDP4A); the indicator
// masks x & 0x80808080 are derived once per chunk into a second shared-memory plane, so the ALU
// pipe (the binding one: half the FMA pipe's rate) sees exactly 2 instructions per compare.  The
// dot product accumulates 128 x matches in one 32-bit register per pair (exact while
// 512 W_j < 2^32).  Tiles of ordinary rectangles end in the candidate test c + f_i + f_j >= s
// (exact corrections follow in finalize.cu) with one append per warp; tiles of accumulated
// rectangles add their partial counts to global counters, thresholded by k2_acc_threshold.
#include <cudaTypedefs.h>

#include <chrono>
#include <cstdio>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "plan.h"

namespace bm {

constexpr int kBM = kTile, kBK = kChunk;
// Tile shapes: 128 x 128 pairs per CTA (8 warps, 2 CTAs per SM, 3 TMA stages) or 128 x 64 (4 warps,
// 4 CTAs per SM, 2 stages) for small or ragged plans; each thread owns an 8 x 8 micro-tile either way.
template <int BN>
struct K2Cfg {
    static constexpr int kThreads = 2 * BN;
    static constexpr int kStages = BN == 128 ? 3 : 2;
    static constexpr int kMinBlocks = BN == 128 ? 2 : 4;
    static constexpr int kStageWords = kBK * (kBM + BN);  // raw words TMA writes per stage
    static constexpr int kStageSmem = 2 * kStageWords;     // + the indicator-mask plane the consumers derive
    static constexpr size_t kSmemBytes = (size_t)kStages * kStageSmem * 4 + kStages * 8;
};
constexpr int kMaxMaps = 48;  // per operand role: 2 x 48 x 128 B of __grid_constant__ parameters
constexpr int kMaxTiledW = 1 << 23;  // 512 * W < 2^32 keeps the 128x-scaled counters exact

struct K2Maps {
    CUtensorMap a[kMaxMaps];  // row operand: box [16 words x 128 items]; classes
    CUtensorMap b[kMaxMaps];  // column operand: box [16 words x BN items]; classes, then virtual copies
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// SWAR compare-and-count step, 4 instructions: acc += 128 * matches.
//   u = (x ^ y) | 0x80808080            LOP3
//   p = u - 0x01010101                  IADD3
//   v = ~p & (xm | ym)                  LOP3 (xm = x & M, ym = y & M from the mask plane; an
//                                             explicit lop3, else ptxas recomputes (x|y)&M per pair)
//   acc = dp4a(v, 0x01010101, acc)      IDP4A: every byte of v is 0x80 or 0
// (tools/swar_ubench.cu: this mix runs at 0.84 of R_int = 32 compares/clk/SM, with or without the
// shared-memory operand loads -- the practical ceiling of the inner loop on B200.)
__device__ __forceinline__ uint32_t swar_step(uint32_t x, uint32_t y, uint32_t xm, uint32_t ym, uint32_t acc) {
    const uint32_t u = (x ^ y) | 0x80808080u;
    const uint32_t p = u - 0x01010101u;
    uint32_t v, r;
    asm("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v) : "r"(p), "r"(xm), "r"(ym));  // ~p & (xm | ym)
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "n"(0x01010101), "r"(acc));
    return r;
}

// The paper's literal formula, used by the simple kernel and the self-test.
__device__ __forceinline__ uint32_t swar_paper(uint32_t x, uint32_t y) {
    uint32_t p = ((x ^ y) | 0x80808080u) - 0x01010101u;
    uint32_t pp = (p ^ 0xFFFFFFFFu) & ((x | y) & 0x80808080u);
    return ((pp >> 7) + (pp >> 15) + (pp >> 23) + (pp >> 31)) & 7u;
}

// ------------------------------------------------------------------ tiled kernel
// Operands of one k step for a thread: 8 row words (x), 8 column words (y) and their masks.
struct Ops {
    uint4 xa, xb, ya, yb, ma, mb, na, nb;
};

// The thread's 8 x 8 micro-tile is four 4 x 4 blocks: bit 0 LL (rows 4tr.., cols 4tc..), bit 1 LH
// (cols BN/2 + 4tc..), bit 2 HL (rows 64 + 4tr..), bit 3 HH.  INC is the set a warp computes for the
// current work item; blocks whose pairs are all invalid (below the diagonal of a diagonal tile, or
// beyond a ragged edge) are skipped, with their operands' loads (block_mask).
constexpr int kLL = 1, kLH = 2, kHL = 4, kHH = 8, kAll = 15;

template <int BN, int INC = kAll>
__device__ __forceinline__ void load_ops(Ops& o, const uint32_t* pa, const uint32_t* pb) {
    // pa = sA + 4 tr + k kBM (row words; masks kStageWords further), pb = sB + 4 tc + k BN
    constexpr int kM = K2Cfg<BN>::kStageWords;  // offset of the mask plane
    if (INC & (kLL | kLH)) {
        o.xa = *reinterpret_cast<const uint4*>(pa);
        o.ma = *reinterpret_cast<const uint4*>(pa + kM);
    }
    if (INC & (kHL | kHH)) {
        o.xb = *reinterpret_cast<const uint4*>(pa + 64);
        o.mb = *reinterpret_cast<const uint4*>(pa + kM + 64);
    }
    if (INC & (kLL | kHL)) {
        o.ya = *reinterpret_cast<const uint4*>(pb);
        o.na = *reinterpret_cast<const uint4*>(pb + kM);
    }
    if (INC & (kLH | kHH)) {
        o.yb = *reinterpret_cast<const uint4*>(pb + BN / 2);
        o.nb = *reinterpret_cast<const uint4*>(pb + kM + BN / 2);
    }
}

// Index i * 8 + j of the q-th pair of the included blocks of INC (blocks in bit order, rows major
// inside a block); constant-folded in the unrolled loops.
template <int INC>
__device__ __forceinline__ constexpr int pair_index(int q) {
    int b = 0;
    for (int t = 0, seen = 0; t < 4; ++t)
        if (INC >> t & 1) {
            if (seen == (q >> 4)) {
                b = t;
                break;
            }
            ++seen;
        }
    return ((b >> 1) * 4 + ((q >> 2) & 3)) * 8 + (b & 1) * 4 + (q & 3);
}

template <int INC>
__device__ __forceinline__ constexpr int n_included() {
    return 16 * ((INC & 1) + (INC >> 1 & 1) + (INC >> 2 & 1) + (INC >> 3 & 1));
}

// The 64 compare-and-counts of one k step, written as a software pipeline over the pairs so
// that every ALU-pipe LOP3 is followed by an FMA-pipe op (IADD, IDP4A): the ALU pipe, which
// binds, can then accept an instruction every other cycle.  Dependent instructions sit kD
// pipeline steps apart (kD = 2: two independent compares between a producer and its consumer).
// asm volatile keeps this order.  (tools/swar_ubench.cu: distance 2 runs 1.5 % faster than 1, 3
// and 4 are slower again; the compiler-scheduled loop is ~4 % slower.)
template <int INC = kAll>
__device__ __forceinline__ void compute_ops(const Ops& o, uint32_t (&acc)[8][8]) {
    constexpr int kD = 2;
    constexpr int N = n_included<INC>();
    const uint32_t x[8] = {o.xa.x, o.xa.y, o.xa.z, o.xa.w, o.xb.x, o.xb.y, o.xb.z, o.xb.w};
    const uint32_t y[8] = {o.ya.x, o.ya.y, o.ya.z, o.ya.w, o.yb.x, o.yb.y, o.yb.z, o.yb.w};
    const uint32_t xm[8] = {o.ma.x, o.ma.y, o.ma.z, o.ma.w, o.mb.x, o.mb.y, o.mb.z, o.mb.w};
    const uint32_t ym[8] = {o.na.x, o.na.y, o.na.z, o.na.w, o.nb.x, o.nb.y, o.nb.z, o.nb.w};
    uint32_t u[64], p[64], v[64];
#pragma unroll
    for (int q = 0; q < N + 3 * kD; ++q) {
        if (q < N) {  // u = (x ^ y) | 0x80808080
            const int e = pair_index<INC>(q);
            asm volatile("lop3.b32 %0, %1, %2, 0x80808080, 0xBE;" : "=r"(u[e]) : "r"(x[e >> 3]), "r"(y[e & 7]));
        }
        if (q >= kD && q - kD < N) {  // p = u - 0x01010101
            const int e = pair_index<INC>(q - kD);
            asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[e]) : "r"(u[e]));
        }
        if (q >= 2 * kD && q - 2 * kD < N) {  // v = ~p & (xm | ym)
            const int e = pair_index<INC>(q - 2 * kD);
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v[e]) : "r"(p[e]), "r"(xm[e >> 3]), "r"(ym[e & 7]));
        }
        if (q >= 3 * kD) {  // acc += 128 * matches
            const int e = pair_index<INC>(q - 3 * kD);
            asm volatile("dp4a.u32.u32 %0, %1, 0x01010101, %0;" : "+r"(acc[e >> 3][e & 7]) : "r"(v[e]));
        }
    }
}

// Blocks of the micro-tile that warp `warp` computes on tile (ti, tj) of rectangle r: a block is
// skipped when all its rows or all its columns lie beyond the rectangle, or -- diagonal
// rectangles, pairs i < j only -- when its smallest row is >= its largest column.
template <int BN>
__device__ __forceinline__ int block_mask(const Rect& r, int ti, int tj, int warp) {
    int inc = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int r0 = ti * kBM + (t >> 1) * 64 + 32 * (warp & 1);          // rows [r0, r0 + 32)
        const int c0 = tj * BN + (t & 1) * (BN / 2) + 16 * (warp >> 1);     // cols [c0, c0 + 16)
        const bool skip = r0 >= r.n_rows || c0 >= r.n_cols || (r.diag && r0 >= c0 + 15);
        if (!skip) inc |= 1 << t;
    }
    return inc;
}

// One k-chunk of the warp's included blocks; pa / pb: the thread's first row / column words.
template <int BN, int INC>
__device__ __forceinline__ void chunk_ops(const uint32_t* pa, const uint32_t* pb, uint32_t (&acc)[8][8]) {
#pragma unroll 1
    for (int k = 0; k < kBK; ++k, pa += kBM, pb += BN) {
        Ops o;
        load_ops<BN, INC>(o, pa, pb);
        compute_ops<INC>(o, acc);
    }
}

// ---- balanced mode for accumulated work items (ragged / diagonal tiles of split-K and virtual
// rectangles).  In the default mapping warp w owns four fixed 32-row x 16-column blocks of the tile
// and skips those with no valid pair; in a ragged tile some warps then own 2 valid blocks and
// others 1 or 0, and the CTA waits for the slowest at every chunk's barrier (C3: 15 % of the warp
// samples).  Accumulated items add partial counts with atomics anyway, so the valid blocks' k-steps
// can be dealt evenly instead: the sequence (valid block, k-step) is cut into one contiguous range
// per warp, i.e. at most 4 units (block, k range) per warp, each held in one of the four 4 x 4
// accumulator slots of the thread's micro-tile.  Slot s covers rows 32 rb + 4 (lane & 7) + i and
// columns 16 cb + 4 (lane >> 3) + j of the tile in acc[(s >> 1) 4 + i][(s & 1) 4 + j].
__device__ __forceinline__ uint32_t bal_unit(int rb, int cb, int klo, int khi) {
    return 0x80000000u | ((uint32_t)rb << 24) | ((uint32_t)cb << 16) | ((uint32_t)klo << 8) | (uint32_t)khi;
}

__device__ __forceinline__ bool block_valid(const Rect& r, int ti, int tj, int tn, int rb, int cb) {
    return k2_block_valid(r.n_rows, r.n_cols, r.diag, ti, tj, tn, rb, cb);
}

// CTA-uniform decision (k2_balance_pays, plan.h); on true, writes this warp's units to slots[0..3]
// (0 = empty).
template <int BN>
__device__ __forceinline__ bool plan_balance(const Rect& r, int ti, int tj, int warp, int lane,
                                             uint32_t* __restrict__ slots) {
    constexpr int NW = BN / 16, NCB = BN / 16;  // warps per CTA; 16-column groups per tile
    if (!k2_balance_pays(r.n_rows, r.n_cols, r.diag, ti, tj, BN)) return false;
    int B = 0;
#pragma unroll 1
    for (int rb = 0; rb < 4; ++rb)
#pragma unroll 1
        for (int cb = 0; cb < NCB; ++cb) B += block_valid(r, ti, tj, BN, rb, cb);
    const int total = 16 * B;
    const int lo = warp * total / NW, hi = (warp + 1) * total / NW;
    int n = 0, bi = 0;
    __syncwarp();  // every lane has read the previous item's slots (its epilogue ran before)
#pragma unroll 1
    for (int rb = 0; rb < 4; ++rb)
#pragma unroll 1
        for (int cb = 0; cb < NCB; ++cb) {
            if (!block_valid(r, ti, tj, BN, rb, cb)) continue;
            const int blo = 16 * bi, klo = max(lo, blo) - blo, khi = min(hi, blo + 16) - blo;
            if (khi > klo && n < 4) {
                if (lane == 0) slots[n] = bal_unit(rb, cb, klo, khi);
                ++n;
            }
            ++bi;
        }
    if (lane == 0)
        for (int q = n; q < 4; ++q) slots[q] = 0u;
    __syncwarp();
    return true;
}

// 16 compare-and-counts of one 4 x 4 block into accumulator slot S (same pipeline as compute_ops).
template <int S>
__device__ __forceinline__ void compute_block(const uint4& xv, const uint4& xmv, const uint4& yv, const uint4& ymv,
                                              uint32_t (&acc)[8][8]) {
    constexpr int kD = 2, N = 16;
    const uint32_t x[4] = {xv.x, xv.y, xv.z, xv.w}, y[4] = {yv.x, yv.y, yv.z, yv.w};
    const uint32_t xm[4] = {xmv.x, xmv.y, xmv.z, xmv.w}, ym[4] = {ymv.x, ymv.y, ymv.z, ymv.w};
    uint32_t u[16], p[16], v[16];
#pragma unroll
    for (int q = 0; q < N + 3 * kD; ++q) {
        if (q < N) asm volatile("lop3.b32 %0, %1, %2, 0x80808080, 0xBE;" : "=r"(u[q]) : "r"(x[q >> 2]), "r"(y[q & 3]));
        if (q >= kD && q - kD < N) asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[q - kD]) : "r"(u[q - kD]));
        if (q >= 2 * kD && q - 2 * kD < N) {
            const int e = q - 2 * kD;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v[e]) : "r"(p[e]), "r"(xm[e >> 2]), "r"(ym[e & 3]));
        }
        if (q >= 3 * kD) {
            const int e = q - 3 * kD;
            asm volatile("dp4a.u32.u32 %0, %1, 0x01010101, %0;"
                         : "+r"(acc[(S >> 1) * 4 + (e >> 2)][(S & 1) * 4 + (e & 3)])
                         : "r"(v[e]));
        }
    }
}

// One k-chunk in balanced mode: each of the warp's units runs its k range on its block.
template <int BN, int S>
__device__ __forceinline__ void chunk_unit(const uint32_t* sA, const uint32_t* sB, uint32_t unit, int lane,
                                           uint32_t (&acc)[8][8]) {
    constexpr int kM = K2Cfg<BN>::kStageWords;
    if (!unit) return;
    const int rb = (unit >> 24) & 3, cb = (unit >> 16) & 15, klo = (unit >> 8) & 31, khi = unit & 31;
    const uint32_t* pa = sA + 32 * rb + 4 * (lane & 7) + klo * kBM;
    const uint32_t* pb = sB + 16 * cb + 4 * (lane >> 3) + klo * BN;
#pragma unroll 1
    for (int k = klo; k < khi; ++k, pa += kBM, pb += BN) {
        const uint4 xv = *reinterpret_cast<const uint4*>(pa), xmv = *reinterpret_cast<const uint4*>(pa + kM);
        const uint4 yv = *reinterpret_cast<const uint4*>(pb), ymv = *reinterpret_cast<const uint4*>(pb + kM);
        compute_block<S>(xv, xmv, yv, ymv, acc);
    }
}

// End of a balanced item: add every slot's partial counts to the rectangle's counters (the
// accumulated epilogue of work_epilogue with per-slot rows and columns).
template <int BN>
__device__ __forceinline__ void bal_epilogue(const Rect& r, int ti, int tj, int lane, const uint32_t* slots,
                                             const uint32_t (&acc)[8][8], uint32_t* __restrict__ cnt) {
    uint32_t* base = cnt + r.cnt_off;
    const int lgR = __ffs(r.R) - 1;  // R is a power of two (widths 3r/4)
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
        const uint32_t unit = slots[sl];
        if (!unit) continue;
        const int rb = (unit >> 24) & 3, cb = (unit >> 16) & 15;
        const int row0 = ti * kBM + 32 * rb + 4 * (lane & 7), col0 = tj * BN + 16 * cb + 4 * (lane >> 3);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int row = row0 + i;
            if (row >= r.n_rows) continue;
            uint32_t* rowp = base + (int64_t)row * r.n_cols_real;
            const uint32_t* a = acc[(sl >> 1) * 4 + i] + (sl & 1) * 4;
            if (r.R >= 4) {  // the 4 columns are 4 virtual columns of one item
                if (col0 >= r.n_cols) continue;
                const uint32_t sum = (a[0] >> 7) + (a[1] >> 7) + (a[2] >> 7) + (a[3] >> 7);
                if (sum) atomicAdd(rowp + (col0 >> lgR), sum);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int col = col0 + j;
                    if (col >= r.n_cols || (r.diag && row >= col)) continue;
                    const uint32_t v = a[j] >> 7;
                    if (v) atomicAdd(rowp + (col >> lgR), v);
                }
            }
        }
    }
}

// Per-CTA stream of k-chunks.  Work items (longest first) are claimed from a global counter by
// thread 0 -- longest-processing-time order, so the CTAs finish within about one short item of
// each other.  The narrow operand's chunk coordinate wraps mod W_a (reading #18).
struct Cursor {
    int w, kc, k1, ka, Wa, ti, tj, ma, mb, first;
    __device__ __forceinline__ void claim(const Rect* rects, const Work* work, int n_work, int* ctr) {
        w = atomicAdd(ctr, 1);
        if (w < n_work) {
            const Work wk = work[w];
            const Rect& r = rects[wk.rect];
            Wa = r.W_a;
            ma = r.map_a;
            mb = r.map_b;
            ti = wk.ti;
            tj = wk.tj;
            kc = wk.k0;
            k1 = wk.k1;
            ka = (int)(((int64_t)kc * kBK) % Wa);
            first = 1;
        }
    }
};

// Thread 0: fill buffer `buf` with the cursor's next chunk (TMA), or post the end marker once.
template <int BN>
__device__ __forceinline__ void issue_next(const K2Maps& prm, Cursor& c, const Rect* rects, const Work* work,
                                           int n_work, int* ctr, uint32_t* stages, int buf, uint64_t* full,
                                           int2* meta, bool& end_sent) {
    using Cfg = K2Cfg<BN>;
    if (c.w < n_work) {
        uint32_t* sA = stages + buf * Cfg::kStageSmem;
        uint32_t* sB = sA + kBK * kBM;
        meta[buf] = make_int2(c.w, c.first);  // published by the mbarrier's release/acquire
        mbar_expect_tx(&full[buf], Cfg::kStageWords * 4);
        tma_load_2d(sA, &prm.a[c.ma], c.ti * kBM, c.ka, &full[buf]);  // B_i[w mod W_i]
        tma_load_2d(sB, &prm.b[c.mb], c.tj * BN, c.kc * kBK, &full[buf]);
        c.first = 0;
        ++c.kc;
        c.ka += kBK;
        if (c.ka == c.Wa) c.ka = 0;
        if (c.kc == c.k1) c.claim(rects, work, n_work, ctr);
    } else if (!end_sent) {
        meta[buf] = make_int2(-1, 1);
        mbar_arrive(&full[buf]);
        end_sent = true;
    }
}

__device__ __forceinline__ void append_candidates(uint64_t mask, int cnt, int lane, const int (&rows)[8],
                                                  const int (&cols)[8], int fa, int fb, const uint32_t (&acc)[8][8],
                                                  Cand* __restrict__ out, unsigned long long* __restrict__ ctr,
                                                  int64_t cap) {
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    unsigned long long base = 0;
    if (lane == 31 && incl > 0) base = atomicAdd(ctr, (unsigned long long)incl);
    base = __shfl_sync(0xffffffffu, base, 31);
    unsigned long long at = base + (unsigned long long)(incl - cnt);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (mask >> (i * 8 + j) & 1) {
                if ((int64_t)at < cap) {
                    Cand cd;
                    cd.i = (uint32_t)(fa + rows[i]);
                    cd.j = (uint32_t)(fb + cols[j]);
                    cd.c = acc[i][j] >> 7;
                    out[at] = cd;
                }
                ++at;
            }
}

// End of a work item: ordinary rectangles test c + f_i + f_j >= thr and append; accumulated ones
// add the partial counts to their counters (4 adjacent virtual columns of one item pre-summed).
template <int BN>
__device__ __forceinline__ void work_epilogue(const Rect& r, int ti, int tj, int tr, int tc, int lane,
                                              const uint32_t (&acc_in)[8][8], uint32_t* __restrict__ cnt,
                                              const int32_t* __restrict__ f, const uint8_t* __restrict__ lw,
                                              uint32_t thr, uint32_t use_f, Cand* __restrict__ out,
                                              unsigned long long* __restrict__ ctr, int64_t cap) {
    int rows[8], cols[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        rows[i] = ti * kBM + (i < 4 ? 4 * tr + i : 64 + 4 * tr + (i - 4));
        cols[i] = tj * BN + (i < 4 ? 4 * tc + i : BN / 2 + 4 * tc + (i - 4));
    }
    if (r.acc) {  // scaled partial counts; k2_acc_threshold divides promoted pairs
        const uint32_t (&acc)[8][8] = acc_in;
        uint32_t* base = cnt + r.cnt_off;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (rows[i] >= r.n_rows) continue;
            uint32_t* row = base + (int64_t)rows[i] * r.n_cols_real;
            if (r.R >= 4) {  // columns 4g..4g+3 are 4 virtual columns of the same item
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    if (cols[4 * g] >= r.n_cols) continue;
                    const uint32_t s = (acc[i][4 * g] >> 7) + (acc[i][4 * g + 1] >> 7) + (acc[i][4 * g + 2] >> 7) +
                                       (acc[i][4 * g + 3] >> 7);
                    if (s) atomicAdd(row + cols[4 * g] / r.R, s);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (cols[j] >= r.n_cols || (r.diag && rows[i] >= cols[j])) continue;
                    const uint32_t s = acc[i][j] >> 7;
                    if (s) atomicAdd(row + cols[j] / r.R, s);
                }
            }
        }
        return;
    }
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = acc_in[i][j];
    if (r.promo) {  // promoted pairs compared K = 2^lgK W_min words: K / max(W_i, W_j) times the count
        int lr[8], lc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            lr[i] = rows[i] < r.n_rows ? (int)__ldg(lw + r.row_first + rows[i]) : 0;
            lc[i] = cols[i] < r.n_cols ? (int)__ldg(lw + r.col_first + cols[i]) : 0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = ((acc[i][j] >> 7) >> (r.lgK - max(lr[i], lc[j]))) << 7;
    }
    uint32_t fr[8], fc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        fr[i] = (use_f && rows[i] < r.n_rows) ? (uint32_t)__ldg(f + r.row_first + rows[i]) : 0u;
        fc[i] = (use_f && cols[i] < r.n_cols) ? (uint32_t)__ldg(f + r.col_first + cols[i]) : 0u;
    }
    uint64_t mask = 0;
    int n = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const bool valid = rows[i] < r.n_rows && cols[j] < r.n_cols && (!r.diag || rows[i] < cols[j]);
            const uint64_t c = acc[i][j] >> 7;
            if (valid && c + fr[i] + fc[j] >= thr) {
                mask |= 1ull << (i * 8 + j);
                ++n;
            }
        }
    append_candidates(mask, n, lane, rows, cols, r.row_first, r.col_first, acc, out, ctr, cap);
}

// 2 BN threads = BN / 16 warps; thread (tr, tc) owns rows {4tr..4tr+3, 64+4tr..+3} x cols {4tc..,
// BN/2+4tc..} of the 128 x BN tile.  Thread 0 also drives TMA: after the per-chunk barrier every
// warp has finished the previous chunk, so that buffer is refilled with the chunk kStages-1 ahead.
template <int BN>
__global__ void __launch_bounds__(K2Cfg<BN>::kThreads, K2Cfg<BN>::kMinBlocks)
    k2_tiled(const __grid_constant__ K2Maps prm, const Rect* __restrict__ rects, const Work* __restrict__ work,
             int n_work, int* work_ctr, uint32_t* __restrict__ cnt, uint32_t* __restrict__ tail_buf, int tail_pieces,
             const int32_t* __restrict__ f, const uint8_t* __restrict__ lw, uint32_t thr, uint32_t use_f,
             Cand* __restrict__ out, unsigned long long* __restrict__ ctr, int64_t cap, int bal_enabled) {
    using Cfg = K2Cfg<BN>;
    constexpr int kStages = Cfg::kStages, kStageSmem = Cfg::kStageSmem, kStageWords = Cfg::kStageWords;
    constexpr int kThreads = Cfg::kThreads;
    extern __shared__ __align__(1024) uint32_t smem_raw[];
    uint32_t* stages = smem_raw;  // keep the shared address space visible to the compiler (LDS, not LD)
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + kStages * kStageSmem);
    __shared__ int2 meta[kStages];
    __shared__ uint32_t bal_slots[kThreads / 32][4];  // balanced-mode units of each warp

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    Cursor pre;  // prefetch cursor (thread 0 only)
    bool end_sent = false;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        pre.claim(rects, work, n_work, work_ctr);
        for (int s = 0; s < kStages - 1; ++s)
            issue_next<BN>(prm, pre, rects, work, n_work, work_ctr, stages, s, full, meta, end_sent);
    }
    __syncthreads();

    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    int cur = -1;
    int inc = kAll;
    bool bal = false;  // the current item runs in balanced mode (CTA-uniform)
    uint32_t* my_slots = bal_slots[warp];
    const bool bal_on = bal_enabled;
    for (uint32_t g = 0;; ++g) {
        const int buf = (int)(g % kStages);
        mbar_wait(&full[buf], (g / kStages) & 1u);
        const int2 mt = meta[buf];
        if (mt.y && cur >= 0) {  // a new work item (or the end) begins: finish the previous one
            const Work wk = work[cur];
            if (wk.tail && bal) {  // a balanced ordinary tile: each slot's counts go where the
                                   // default mapping keeps that pair (thread 32 w' + lane, block (h, hc))
                uint32_t* slice = tail_buf + (int64_t)((wk.tail - 1) / tail_pieces) * (kBM * BN);
#pragma unroll
                for (int sl = 0; sl < 4; ++sl) {
                    const uint32_t unit = my_slots[sl];
                    if (!unit) continue;
                    const int rb = (unit >> 24) & 3, cb = (unit >> 16) & 15;
                    const int w2 = (rb & 1) | ((cb % (BN / 32)) << 1), h = rb >> 1, hc = cb / (BN / 32);
                    uint32_t* dst = slice + 4 * (32 * w2 + lane);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t v = acc[(sl >> 1) * 4 + i][(sl & 1) * 4 + j];
                            if (v)
                                asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(
                                                 dst + (int64_t)((2 * (4 * h + i) + hc) * kThreads) * 4 + j),
                                             "r"(v)
                                             : "memory");
                        }
                }
            } else if (wk.tail) {  // a piece of a cut tail tile: partial counts added (red.global.add, in
                            // L2) into its tile's one zeroed slice, laid out as 16 uint4 planes of
                            // kThreads (coalesced loads in k2_tail_threshold); one slice per tile
                            // instead of one per piece keeps the tail's writes in L2
                uint32_t* dst = tail_buf + (int64_t)((wk.tail - 1) / tail_pieces) * (kBM * BN) + 4 * threadIdx.x;
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (acc[i][j])
                            asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(
                                             dst + (int64_t)((2 * i + (j >> 2)) * kThreads) * 4 + (j & 3)),
                                         "r"(acc[i][j])
                                         : "memory");
            } else if (bal) {
                bal_epilogue<BN>(rects[wk.rect], wk.ti, wk.tj, lane, my_slots, acc, cnt);
            } else {
                work_epilogue<BN>(rects[wk.rect], wk.ti, wk.tj, tr, tc, lane, acc, cnt, f, lw, thr, use_f, out,
                                  ctr, cap);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0;
        }
        if (mt.x < 0) break;
        if (mt.y) {
            // ragged edge and diagonal tiles: blocks of pairs that are all invalid are skipped,
            // leaving their issue slots to the other CTA
            const Work wk = work[mt.x];
            const Rect& rr = rects[wk.rect];
            inc = block_mask<BN>(rr, wk.ti, wk.tj, warp);
            bal = bal_on && (rr.acc || wk.tail) && plan_balance<BN>(rr, wk.ti, wk.tj, warp, lane, my_slots);
        }
        cur = mt.x;
        uint32_t* sA = stages + buf * kStageSmem;
        {  // derive the indicator-mask plane x & 0x80808080 once per chunk (not once per thread)
            const uint4* src = reinterpret_cast<const uint4*>(sA);
            uint4* dst = reinterpret_cast<uint4*>(sA + kStageWords);
#pragma unroll
            for (int q = 0; q < kStageWords / 4 / kThreads; ++q) {
                uint4 v = src[threadIdx.x + kThreads * q];
                v.x &= 0x80808080u;
                v.y &= 0x80808080u;
                v.z &= 0x80808080u;
                v.w &= 0x80808080u;
                dst[threadIdx.x + kThreads * q] = v;
            }
        }
        __syncthreads();  // masks visible; every warp is done with the previous chunk's buffer
        if (threadIdx.x == 0)
            issue_next<BN>(prm, pre, rects, work, n_work, work_ctr, stages, (int)((g + kStages - 1) % kStages),
                           full, meta, end_sent);
        const uint32_t* pa = sA + 4 * tr;
        const uint32_t* pb = sA + kBK * kBM + 4 * tc;
        if (inc == kAll && !bal) {  // the common case first: one test on the hot path
            chunk_ops<BN, kAll>(pa, pb, acc);
        } else if (bal) {
            const uint32_t* sB = sA + kBK * kBM;
            chunk_unit<BN, 0>(sA, sB, my_slots[0], lane, acc);
            chunk_unit<BN, 1>(sA, sB, my_slots[1], lane, acc);
            chunk_unit<BN, 2>(sA, sB, my_slots[2], lane, acc);
            chunk_unit<BN, 3>(sA, sB, my_slots[3], lane, acc);
        } else {
            switch (inc) {  // the reachable block sets; any other non-empty set computes all four
                case 0: break;
                case kLL | kLH | kHH: chunk_ops<BN, kLL | kLH | kHH>(pa, pb, acc); break;  // diagonal tiles
                case kLL | kLH: chunk_ops<BN, kLL | kLH>(pa, pb, acc); break;
                case kLH: chunk_ops<BN, kLH>(pa, pb, acc); break;
                case kLL | kHL: chunk_ops<BN, kLL | kHL>(pa, pb, acc); break;
                case kLL: chunk_ops<BN, kLL>(pa, pb, acc); break;
                default: chunk_ops<BN, kAll>(pa, pb, acc); break;
            }
        }
    }
}

// Cut tail tiles: one CTA per tile sums its pieces' partial counts (same thread mapping as
// k2_tiled) and runs the ordinary epilogue -- candidate test c + f_i + f_j >= s and append.
template <int BN>
__global__ void __launch_bounds__(K2Cfg<BN>::kThreads) k2_tail_threshold(const TailTile* __restrict__ tails, int pieces,
                                                              const Rect* __restrict__ rects,
                                                              const uint32_t* __restrict__ tail_buf,
                                                              const int32_t* __restrict__ f,
                                                              const uint8_t* __restrict__ lw, uint32_t thr,
                                                              uint32_t use_f, Cand* __restrict__ out,
                                                              unsigned long long* __restrict__ ctr, int64_t cap) {
    const TailTile t = tails[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int p = 0; p < pieces; ++p) {
        const uint4* src =
            reinterpret_cast<const uint4*>(tail_buf + (int64_t)(blockIdx.x * pieces + p) * (kBM * BN)) + threadIdx.x;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 a = src[(2 * i) * K2Cfg<BN>::kThreads], b = src[(2 * i + 1) * K2Cfg<BN>::kThreads];
            acc[i][0] += a.x;
            acc[i][1] += a.y;
            acc[i][2] += a.z;
            acc[i][3] += a.w;
            acc[i][4] += b.x;
            acc[i][5] += b.y;
            acc[i][6] += b.z;
            acc[i][7] += b.w;
        }
    }
    work_epilogue<BN>(rects[t.rect], t.ti, t.tj, tr, tc, lane, acc, nullptr, f, lw, thr, use_f, out, ctr, cap);
}

// Accumulated rectangles: the counters of every owned tile row, spread over a 2-D grid (y: tile
// row, x: chunks of its 128 x n_cols counters, columns fastest: coalesced), candidate test on the
// summed counts, one output cursor atomic per warp.  (One CTA per tile row took 235 us on C1,
// whose whole diagonal rectangle is split along k: 8 tile rows x 128 x 998 counters.)
constexpr int kAccPerThread = 8;
__global__ void __launch_bounds__(256) k2_acc_threshold(const AccUnit* __restrict__ units, int n_units,
                                                        const Rect* __restrict__ rects,
                                                        const uint32_t* __restrict__ cnt,
                                                        const int32_t* __restrict__ f,
                                                        const uint8_t* __restrict__ lw, uint32_t thr, uint32_t use_f,
                                                        Cand* __restrict__ out, unsigned long long* __restrict__ ctr,
                                                        int64_t cap) {
    const int lane = threadIdx.x & 31;
    for (int ui = blockIdx.y; ui < n_units; ui += gridDim.y) {
        const AccUnit u = units[ui];
        const Rect& r = rects[u.rect];
        const int r0 = u.ti * kTile;
        const int nr = min(kTile, r.n_rows - r0);
        const int ncol = r.n_cols_real;
        const int total = nr * ncol;
        // warp-uniform trip count (ballots below)
        for (int base = blockIdx.x * blockDim.x * kAccPerThread; base < total;
             base += gridDim.x * blockDim.x * kAccPerThread) {
#pragma unroll
            for (int q = 0; q < kAccPerThread; ++q) {
                const int e = base + q * blockDim.x + threadIdx.x;
                bool take = false;
                int row = 0, col = 0;
                uint32_t c = 0;
                if (e < total) {
                    row = r0 + e / ncol;
                    col = e - (e / ncol) * ncol;
                    if (!r.diag || col > row) {
                        c = cnt[r.cnt_off + (int64_t)row * ncol + col];
                        if (r.promo) c >>= r.lgK - max((int)lw[r.row_first + row], (int)lw[r.col_first + col]);
                        uint64_t t = c;
                        if (use_f) t += (uint32_t)f[r.row_first + row] + (uint32_t)f[r.col_first + col];
                        take = t >= thr;
                    }
                }
                const unsigned mask = __ballot_sync(0xFFFFFFFFu, take);
                if (!mask) continue;
                unsigned long long at = 0;
                const int leader = __ffs(mask) - 1;
                if (lane == leader) at = atomicAdd(ctr, (unsigned long long)__popc(mask));
                at = __shfl_sync(0xFFFFFFFFu, at, leader) + __popc(mask & ((1u << lane) - 1));
                if (take && (int64_t)at < cap) {
                    Cand cd;
                    cd.i = (uint32_t)(r.row_first + row);
                    cd.j = (uint32_t)(r.col_first + col);
                    cd.c = c;
                    out[at] = cd;
                }
            }
        }
    }
}

// Virtual copy of class b for period W_a: dst[k * vpad + v] = word (rep W_a + k) of item j,
// v = j R + rep; padding columns are ⊥ words.
__global__ void k_virtualize(const uint32_t* __restrict__ src, int32_t src_npad, int32_t n_b, int32_t W_a, int32_t R,
                             int32_t vpad, uint32_t* __restrict__ dst) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)W_a * vpad) return;
    const int k = (int)(idx / vpad);
    const int v = (int)(idx - (int64_t)k * vpad);
    uint32_t word = kNullWord;
    if (v < n_b * R) {
        const int j = v / R, rep = v - (v / R) * R;
        word = src[((int64_t)rep * W_a + k) * src_npad + j];
    }
    dst[idx] = word;
}

// Promoted group: dst[w * n_pad + c] = word (w mod W_k) of item c, taken from its own class k's
// block (B'[w] = B[w mod W_k], W_k | W); padding columns are ⊥ words.
constexpr int kMaxPromoMembers = 32;
struct PromoSrc {
    int32_t n_members, W, n, n_pad;
    int64_t word_off[kMaxPromoMembers];
    int32_t c0[kMaxPromoMembers + 1], W_k[kMaxPromoMembers], npad_k[kMaxPromoMembers];
};

__global__ void k_promote(const uint32_t* __restrict__ arena, const __grid_constant__ PromoSrc ps,
                          uint32_t* __restrict__ dst) {
    const int64_t total = (int64_t)ps.W * ps.n_pad;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(idx / ps.n_pad);
        const int c = (int)(idx - (int64_t)w * ps.n_pad);
        uint32_t word = kNullWord;
        if (c < ps.n) {
            int k = 0;
            while (c >= ps.c0[k + 1]) ++k;
            word = arena[ps.word_off[k] + (int64_t)(w % ps.W_k[k]) * ps.npad_k[k] + (c - ps.c0[k])];
        }
        dst[idx] = word;
    }
}

// ------------------------------------------------------------------ simple kernel (one thread per pair)
struct SimpleClass {
    int64_t word_off;
    int32_t n, n_pad, W, first;
};

__global__ void __launch_bounds__(256) k2_simple(const uint32_t* __restrict__ arena,
                                                 const SimpleClass* __restrict__ cls,
                                                 const int4* __restrict__ tiles,
                                                 const int32_t* __restrict__ f, uint32_t thr,
                                                 uint32_t use_f, Cand* __restrict__ out,
                                                 unsigned long long* __restrict__ ctr, int64_t cap) {
    const int4 td = tiles[blockIdx.x];
    const SimpleClass A = cls[td.x], B = cls[td.y];
    const int row = td.z * 16 + threadIdx.y, col = td.w * 16 + threadIdx.x;
    const bool valid = row < A.n && col < B.n && (td.x != td.y || row < col);
    if (!valid) return;
    const uint32_t* pa = arena + A.word_off + row;
    const uint32_t* pb = arena + B.word_off + col;
    uint32_t c = 0;
    int wa = 0;
    for (int w = 0; w < B.W; ++w) {
        c += swar_paper(pa[(int64_t)wa * A.n_pad], pb[(int64_t)w * B.n_pad]);  // B_i[w mod W_i]
        if (++wa == A.W) wa = 0;
    }
    uint64_t tot = c;
    if (use_f) tot += (uint32_t)f[A.first + row] + (uint32_t)f[B.first + col];
    if (tot >= thr) {
        unsigned long long at = atomicAdd(ctr, 1ull);
        if ((int64_t)at < cap) {
            Cand cd;
            cd.i = (uint32_t)(A.first + row);
            cd.j = (uint32_t)(B.first + col);
            cd.c = c;
            out[at] = cd;
        }
    }
}

__global__ void k_swar_selftest(const uint32_t* __restrict__ x, const uint32_t* __restrict__ y, int64_t n,
                                uint32_t* __restrict__ out, uint32_t one) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t a = x[k], b = y[k];
    out[k] = swar_step(a, b, a & 0x80808080u, b & 0x80808080u, 0u) >> 7;
    out[n + k] = swar_paper(a, b);
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {  // thread-safe one-time lookup
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        cudaGetLastError();
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}

void plan_tiles(const std::vector<ClassInfo>& cls, int tile_m, int part, int n_parts, TileList* out) {
    struct T {
        int4 t;
        int64_t cost;
    };
    std::vector<T> all;
    const int C = (int)cls.size();
    for (int a = 0; a < C; ++a) {
        const int ta = (cls[a].n + tile_m - 1) / tile_m;
        for (int b = a; b < C; ++b) {
            const int tb = (cls[b].n + tile_m - 1) / tile_m;
            const int64_t cost = (int64_t)tile_m * tile_m * cls[b].W;
            for (int i = 0; i < ta; ++i)
                for (int j = (a == b ? i : 0); j < tb; ++j) all.push_back({make_int4(a, b, i, j), cost});
        }
    }
    // longest first (P:460-461 width order makes equal costs contiguous); deal round-robin
    std::stable_sort(all.begin(), all.end(), [](const T& x, const T& y) { return x.cost > y.cost; });
    out->tiles.clear();
    out->work = 0;
    for (size_t k = 0; k < all.size(); ++k)
        if ((int)(k % (size_t)n_parts) == part) {
            out->tiles.push_back(all[k].t);
            out->work += all[k].cost;
        }
}

static batmap_status ensure_cand(batmap_collection* h, int64_t need, cudaStream_t st) {
    return ensure(&h->cand_d, &h->cand_cap, need, st);
}

static bool env_off(const char* name) {
    const char* e = getenv(name);
    return e && e[0] == '0';
}

static batmap_status encode_map(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, const uint32_t* base,
                                int64_t n_pad, int64_t W, int box_items) {
    cuuint64_t dims[2] = {(cuuint64_t)n_pad, (cuuint64_t)W};
    cuuint64_t strides[1] = {(cuuint64_t)n_pad * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_items, (cuuint32_t)kBK};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return BATMAP_E_CUDA;
    }
    return BATMAP_OK;
}

static batmap_status run_simple(batmap_collection* h, const Selection& sel, uint32_t threshold, int part, int n_parts,
                                uint32_t use_f, cudaStream_t st, int64_t* n_cand) {
    TileList tl;
    plan_tiles(sel.classes, 16, part, n_parts, &tl);
    const int64_t n_tiles = (int64_t)tl.tiles.size();
    int64_t wc = 0;
    for (const int4& t : tl.tiles) {
        const ClassInfo &A = sel.classes[t.x], &B = sel.classes[t.y];
        const int64_t rows = std::min<int64_t>(16, A.n - (int64_t)t.z * 16);
        const int64_t cols = std::min<int64_t>(16, B.n - (int64_t)t.w * 16);
        wc += ((t.x == t.y && t.z == t.w) ? rows * (rows - 1) / 2 : rows * cols) * B.W;
    }
    h->stats.word_compares = wc;
    h->stats.tile_compares = tl.work;
    h->stats.k2_kind = 2;
    h->stats.k2_grid = (int32_t)n_tiles;
    if (n_tiles == 0) return BATMAP_OK;
    std::vector<SimpleClass> sc(sel.classes.size());
    for (size_t a = 0; a < sel.classes.size(); ++a)
        sc[a] = {sel.classes[a].word_off, sel.classes[a].n, sel.classes[a].n_pad, sel.classes[a].W,
                 (int32_t)sel.classes[a].first};
    int4* tiles_d = nullptr;
    SimpleClass* scls_d = nullptr;
    Scratch scratch(st);
    scratch.own(&tiles_d);
    scratch.own(&scls_d);
    BM_TRY(dalloc_t(&tiles_d, n_tiles, st));
    BM_TRY(dalloc_t(&scls_d, (int64_t)sc.size(), st));
    BM_CUDA(cudaMemcpyAsync(tiles_d, tl.tiles.data(), n_tiles * sizeof(int4), cudaMemcpyHostToDevice, st));
    BM_CUDA(cudaMemcpyAsync(scls_d, sc.data(), sc.size() * sizeof(SimpleClass), cudaMemcpyHostToDevice, st));
    batmap_status rc = BATMAP_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {
        BM_CUDA(cudaMemsetAsync(h->ctr_d, 0, sizeof(unsigned long long), st));
        rec(h, EV_K20, st);
        k2_simple<<<(unsigned)n_tiles, dim3(16, 16), 0, st>>>(sel.arena, scls_d, tiles_d, sel.f, threshold, use_f,
                                                             h->cand_d, h->ctr_d, h->cand_cap);
        rec(h, EV_K21, st);
        h->launches += 1;
        BM_CUDA(cudaGetLastError());
        unsigned long long cnt = 0;
        BM_TRY(read_scalar(st, h->ctr_d, &cnt));
        *n_cand = (int64_t)cnt;
        if ((int64_t)cnt <= h->cand_cap) break;
        rc = ensure_cand(h, (int64_t)cnt, st);
        if (rc != BATMAP_OK) break;
    }
    return rc;
}

static int min_blocks(int tn) { return tn == 128 ? K2Cfg<128>::kMinBlocks : K2Cfg<64>::kMinBlocks; }

static int env_tn() {  // BATMAP_K2_TN: 0 = the planner's choice
    const char* e = getenv("BATMAP_K2_TN");
    return e ? atoi(e) : 0;
}

struct K2Prepared {
    int part = -1, n_parts = -1;
    int tn = kTile;       // tile width of the plan
    int tn_env = 0;       // BATMAP_K2_TN when planned
    bool promote = true;  // planned with class promotion (BATMAP_K2_PROMOTE)
    Plan pl;
    K2Maps* prm = nullptr;
    Rect* rects_d = nullptr;
    Work* work_d = nullptr;
    AccUnit* units_d = nullptr;
    TailTile* tails_d = nullptr;
    uint32_t* virt_d = nullptr;
    uint32_t* promo_d = nullptr;  // promoted class blocks
    uint8_t* lw_d = nullptr;      // per selection position: log2(W_i / W_min), if any promotion
};

void release_k2(K2Prepared* kp, cudaStream_t st) {
    if (!kp) return;
    delete kp->prm;
    kp->prm = nullptr;
    dfree(kp->rects_d, st);
    dfree(kp->work_d, st);
    dfree(kp->units_d, st);
    dfree(kp->tails_d, st);
    dfree(kp->virt_d, st);
    dfree(kp->promo_d, st);
    dfree(kp->lw_d, st);
    kp->promo_d = nullptr;
    kp->lw_d = nullptr;
    kp->tails_d = nullptr;
    kp->rects_d = nullptr;
    kp->work_d = nullptr;
    kp->units_d = nullptr;
    kp->virt_d = nullptr;
}

void destroy_k2(K2Prepared* kp, cudaStream_t st) {
    release_k2(kp, st);
    delete kp;
}

// Host planning + device copies of the plan + tensor maps (no dependence on the arena contents).
// Host half of the plan: tile width and work list (pure host computation, no device calls; the build
// runs it on a worker thread while the K1 kernels execute).
void plan_k2_host(const std::vector<ClassInfo>& classes, int num_sms, int part, int n_parts, K2Prepared* kp) {
    kp->part = part;
    kp->n_parts = n_parts;
    const bool promote = !env_off("BATMAP_K2_PROMOTE");
    const bool virt = !env_off("BATMAP_K2_VIRTUAL");
    kp->promote = promote;
    kp->tn = choose_tn(classes, virt, promote);
    kp->tn_env = env_tn();
    const int grid_cap = min_blocks(kp->tn) * num_sms;
    plan_work(classes, part, n_parts, grid_cap, virt, !env_off("BATMAP_K2_SPLIT"), promote, &kp->pl, kp->tn);
    if ((int)kp->pl.eff.size() > kMaxMaps || (int)(kp->pl.eff.size() + kp->pl.virt.size()) > kMaxMaps)
        plan_work(classes, part, n_parts, grid_cap, false, true, promote, &kp->pl, kp->tn);
}

// Device half: scratch copies, tensor maps, and the plan's upload.
namespace {
struct MTrace {  // BATMAP_TRACE=2: timestamps inside the plan upload (diagnostics)
    bool on;
    std::chrono::steady_clock::time_point last;
    MTrace() {
        const char* e = getenv("BATMAP_TRACE");
        on = e && e[0] == '2';
        last = std::chrono::steady_clock::now();
    }
    void mark(const char* w) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[batmap upload] %-22s +%9.3f ms\n", w, std::chrono::duration<double, std::milli>(now - last).count());
        last = now;
    }
};
}  // namespace

static batmap_status materialize_k2(batmap_collection* h, const Selection& sel, cudaStream_t st, K2Prepared* kp) {
    MTrace mt;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return BATMAP_E_CUDA;
    }
    const Plan& pl = kp->pl;
    const int C = (int)pl.eff.size();
    if (pl.work.empty()) return BATMAP_OK;
    if (pl.virt_words) BM_TRY(dalloc_t(&kp->virt_d, pl.virt_words, st));
    mt.mark("virt alloc");
    if (pl.promo_words) {
        for (const PromoCopy& pc : pl.promo)
            if (pc.cls_hi - pc.cls_lo + 1 > kMaxPromoMembers) {
                set_error("promoted group of %d classes", pc.cls_hi - pc.cls_lo + 1);
                return BATMAP_E_INVALID;
            }
        BM_TRY(dalloc_t(&kp->promo_d, pl.promo_words, st));
        std::vector<uint8_t> lw((size_t)sel.n_sel, 0);
        for (const ClassInfo& c : sel.classes)
            for (int64_t q = 0; q < c.n; ++q) lw[(size_t)(c.first + q)] = (uint8_t)lg_ratio(c.W, sel.classes[0].W);
        BM_TRY(dalloc_t(&kp->lw_d, sel.n_sel, st));
        BM_CUDA(cudaMemcpyAsync(kp->lw_d, lw.data(), lw.size(), cudaMemcpyHostToDevice, st));
        BM_CUDA(cudaStreamSynchronize(st));  // lw is a host temporary
    }
    mt.mark("promo");
    kp->prm = new K2Maps();
    for (int a = 0; a < C; ++a) {  // row role (box 128 items) and column role (box tn items)
        const uint32_t* base = pl.eff_promo[a] >= 0 ? kp->promo_d : sel.arena;
        BM_TRY(encode_map(enc, &kp->prm->a[a], base + pl.eff[a].word_off, pl.eff[a].n_pad, pl.eff[a].W, kBM));
        BM_TRY(encode_map(enc, &kp->prm->b[a], base + pl.eff[a].word_off, pl.eff[a].n_pad, pl.eff[a].W, kp->tn));
    }
    for (size_t k = 0; k < pl.virt.size(); ++k)
        BM_TRY(encode_map(enc, &kp->prm->b[C + k], kp->virt_d + pl.virt[k].dst_word_off, pl.virt[k].vpad,
                          pl.virt[k].W_a, kp->tn));
    mt.mark("tensor maps");
    BM_TRY(dalloc_t(&kp->rects_d, (int64_t)pl.rects.size(), st));
    BM_TRY(dalloc_t(&kp->work_d, (int64_t)pl.work.size(), st));
    BM_TRY(dalloc_t(&kp->units_d, (int64_t)std::max<size_t>(pl.units.size(), 1), st));
    if (!pl.tails.empty()) BM_TRY(dalloc_t(&kp->tails_d, (int64_t)pl.tails.size(), st));
    // the plan goes up through pinned staging: a pageable copy would wait for the build's kernels
    // already queued on the stream (C4: 7.6 MB of work items behind ~2 ms of K1)
    struct Up {
        void* dst;
        const void* src;
        size_t bytes;
    };
    const Up ups[4] = {{kp->rects_d, pl.rects.data(), pl.rects.size() * sizeof(Rect)},
                       {kp->work_d, pl.work.data(), pl.work.size() * sizeof(Work)},
                       {kp->units_d, pl.units.data(), pl.units.size() * sizeof(AccUnit)},
                       {kp->tails_d, pl.tails.data(), pl.tails.size() * sizeof(TailTile)}};
    size_t total = 0;
    for (const Up& u : ups) total += (u.bytes + 15) / 16 * 16;
    mt.mark("plan allocs");
    char* pin = static_cast<char*>(host_staging(total, 1));
    mt.mark("staging");
    size_t at = 0;
    for (const Up& u : ups) {
        if (!u.bytes) continue;
        const void* from = u.src;
        if (pin) {
            memcpy(pin + at, u.src, u.bytes);
            from = pin + at;
            at += (u.bytes + 15) / 16 * 16;
        }
        BM_CUDA(cudaMemcpyAsync(u.dst, from, u.bytes, cudaMemcpyHostToDevice, st));
    }
    mt.mark("copies queued");
    return BATMAP_OK;
}

// Called by batmap_build once the classes are known: plan the full selection for (part, n_parts).
batmap_status prepare_k2(batmap_collection* h, const Selection& sel, int part, int n_parts, cudaStream_t st,
                         K2Prepared* kp) {
    plan_k2_host(sel.classes, h->num_sms, part, n_parts, kp);
    return materialize_k2(h, sel, st, kp);
}

bool full_k2_plannable(const batmap_collection* h) {
    if (h->n < 2 || (int)h->classes.size() > kMaxMaps) return false;
    for (const ClassInfo& c : h->classes)
        if (c.W % kBK != 0 || c.W >= kMaxTiledW || c.W < kBK) return false;
    return true;
}

K2Prepared* new_k2_host_plan(const std::vector<ClassInfo>& classes, int num_sms, int part, int n_parts) {
    K2Prepared* kp = new K2Prepared();
    plan_k2_host(classes, num_sms, part, n_parts, kp);
    return kp;
}

// The plan of the full selection, from a host plan made beforehand (hp, owned from here on) or now.
batmap_status prepare_full_k2(batmap_collection* h, int part, int n_parts, cudaStream_t st, K2Prepared* hp) {
    if (!full_k2_plannable(h)) {
        if (hp) destroy_k2(hp, st);
        return BATMAP_OK;
    }
    Selection sel;
    sel.classes = h->classes;
    sel.arena = h->arena_d;
    sel.n_sel = h->n;
    K2Prepared* kp = hp ? hp : new K2Prepared();
    batmap_status rc = hp ? materialize_k2(h, sel, st, kp) : prepare_k2(h, sel, part, n_parts, st, kp);
    if (rc != BATMAP_OK) {
        destroy_k2(kp, st);
        return rc;
    }
    if (h->k2prep) destroy_k2(h->k2prep, st);
    h->k2prep = kp;
    return BATMAP_OK;
}

batmap_status run_intersect(batmap_collection* h, const Selection& sel, uint32_t threshold, int part,
                            int n_parts, uint32_t flags, cudaStream_t st, int64_t* n_cand) {
    *n_cand = 0;
    if (sel.n_sel < 2) return BATMAP_OK;
    if (!h->ctr_d) BM_TRY(dalloc_t(&h->ctr_d, 2, st));
    if (h->cand_cap == 0) BM_TRY(ensure_cand(h, std::max<int64_t>(1 << 20, sel.n_sel * 16), st));
    const uint32_t use_f = (flags & BATMAP_PAIRS_RAW) ? 0u : 1u;
    bool simple = (flags & BATMAP_PAIRS_SIMPLE) != 0;
    for (const ClassInfo& c : sel.classes)
        if (c.W % kBK != 0 || c.W >= kMaxTiledW || c.W < kBK) simple = true;
    PFN_cuTensorMapEncodeTiled_v12000 enc = simple ? nullptr : tensor_map_encoder();
    if (!enc) simple = true;
    const int C = (int)sel.classes.size();
    if (C > kMaxMaps) simple = true;
    if (simple) return run_simple(h, sel, threshold, part, n_parts, use_f, st, n_cand);

    // the plan of the full selection is prepared (host planning, H2D, tensor maps) while the build
    // kernels run, and reused; item subsets are planned here
    K2Prepared* kp = nullptr;
    K2Prepared local;
    if (!sel.sel2pos && h->k2prep && h->k2prep->part == part && h->k2prep->n_parts == n_parts &&
        h->k2prep->promote == !env_off("BATMAP_K2_PROMOTE") && h->k2prep->tn_env == env_tn()) {
        kp = h->k2prep;
    } else {
        const batmap_status prc = prepare_k2(h, sel, part, n_parts, st, &local);
        if (prc != BATMAP_OK) {
            release_k2(&local, st);
            return prc;
        }
        kp = &local;
    }
    // an item subset's plan buffers (promoted / virtualised copies can be hundreds of MB) are
    // released on every return path, the BM_CUDA / BM_TRY early returns included
    struct LocalPlanGuard {
        K2Prepared* p;
        cudaStream_t st;
        ~LocalPlanGuard() {
            if (p) release_k2(p, st);  // idempotent
        }
    } local_guard{kp == &local ? &local : nullptr, st};
    const Plan& pl = kp->pl;
    const int tn = kp->tn;
    const int grid_cap = min_blocks(tn) * h->num_sms;
    const int64_t n_work = (int64_t)pl.work.size();
    h->stats.word_compares = pl.word_compares;
    h->stats.tile_compares = pl.tile_compares;
    h->stats.k2_kind = 1;
    h->stats.k2_grid = (int32_t)std::min<int64_t>(n_work, grid_cap);
    h->stats.k2_tile_cols = tn;
    if (n_work == 0) {
        if (kp == &local) release_k2(&local, st);
        return BATMAP_OK;
    }
    // promoted groups, then virtual copies of the wide classes of skinny rectangles (after the build
    // kernels wrote the arena; a virtual copy may read a promoted block)
    for (const PromoCopy& pc : pl.promo) {
        PromoSrc ps{};
        ps.n_members = pc.cls_hi - pc.cls_lo + 1;
        ps.W = pc.W;
        ps.n = pc.n;
        ps.n_pad = pc.n_pad;
        int32_t c0 = 0;
        for (int k = 0; k < ps.n_members; ++k) {
            const ClassInfo& A = sel.classes[pc.cls_lo + k];
            ps.word_off[k] = A.word_off;
            ps.c0[k] = c0;
            ps.W_k[k] = A.W;
            ps.npad_k[k] = A.n_pad;
            c0 += A.n;
        }
        ps.c0[ps.n_members] = c0;
        const int64_t cnt = (int64_t)pc.W * pc.n_pad;
        const unsigned blocks = (unsigned)std::min<int64_t>((cnt + 255) / 256, 8 * h->num_sms);
        k_promote<<<blocks, 256, 0, st>>>(sel.arena, ps, kp->promo_d + pc.dst_word_off);
        h->launches += 1;
    }
    for (const VirtCopy& v : pl.virt) {
        const ClassInfo& B = pl.eff[v.cls_b];
        const uint32_t* base = pl.eff_promo[v.cls_b] >= 0 ? kp->promo_d : sel.arena;
        const int64_t cnt = (int64_t)v.W_a * v.vpad;
        k_virtualize<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(base + B.word_off, B.n_pad, B.n, v.W_a, v.R,
                                                                    v.vpad, kp->virt_d + v.dst_word_off);
        h->launches += 1;
    }
    if (pl.cnt_entries) BM_TRY(ensure(&h->cnt_d, &h->cnt_cap, pl.cnt_entries, st));
    const int64_t tail_words = (int64_t)pl.tails.size() * kBM * tn;  // one slice per cut tail tile
    if (tail_words) BM_TRY(ensure(&h->tail_d, &h->tail_cap, tail_words, st));
    // per device (no process-wide flag)
    if (tn == 128)
        BM_CUDA(cudaFuncSetAttribute(k2_tiled<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)K2Cfg<128>::kSmemBytes));
    else
        BM_CUDA(cudaFuncSetAttribute(k2_tiled<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)K2Cfg<64>::kSmemBytes));
    const K2Maps* prm = kp->prm;
    Rect* rects_d = kp->rects_d;
    Work* work_d = kp->work_d;
    AccUnit* units_d = kp->units_d;
    batmap_status rc = BATMAP_OK;
    int* work_ctr = reinterpret_cast<int*>(h->ctr_d + 1);
    const int grid = (int)std::min<int64_t>(n_work, grid_cap);
    const int bal_on = env_off("BATMAP_K2_BALANCE") ? 0 : 1;  // balanced accumulated items (test switch)
    for (int attempt = 0; attempt < 2; ++attempt) {
        BM_CUDA(cudaMemsetAsync(h->ctr_d, 0, 2 * sizeof(unsigned long long), st));  // [1] = work counter
        if (pl.cnt_entries) BM_CUDA(cudaMemsetAsync(h->cnt_d, 0, pl.cnt_entries * sizeof(uint32_t), st));
        if (tail_words) BM_CUDA(cudaMemsetAsync(h->tail_d, 0, tail_words * sizeof(uint32_t), st));
        rec(h, EV_K20, st);
        if (tn == 128)
            k2_tiled<128><<<grid, K2Cfg<128>::kThreads, K2Cfg<128>::kSmemBytes, st>>>(
                *prm, rects_d, work_d, (int)n_work, work_ctr, h->cnt_d, h->tail_d, std::max(pl.tail_pieces, 1), sel.f,
                kp->lw_d, threshold, use_f,
                h->cand_d, h->ctr_d, h->cand_cap, bal_on);
        else
            k2_tiled<64><<<grid, K2Cfg<64>::kThreads, K2Cfg<64>::kSmemBytes, st>>>(
                *prm, rects_d, work_d, (int)n_work, work_ctr, h->cnt_d, h->tail_d, std::max(pl.tail_pieces, 1), sel.f,
                kp->lw_d, threshold, use_f,
                h->cand_d, h->ctr_d, h->cand_cap, bal_on);
        rec(h, EV_K21, st);
        h->launches += 1;
        if (!pl.tails.empty()) {
            if (tn == 128)
                k2_tail_threshold<128><<<(unsigned)pl.tails.size(), K2Cfg<128>::kThreads, 0, st>>>(
                    kp->tails_d, 1, rects_d, h->tail_d, sel.f, kp->lw_d, threshold, use_f, h->cand_d,
                    h->ctr_d, h->cand_cap);
            else
                k2_tail_threshold<64><<<(unsigned)pl.tails.size(), K2Cfg<64>::kThreads, 0, st>>>(
                    kp->tails_d, 1, rects_d, h->tail_d, sel.f, kp->lw_d, threshold, use_f, h->cand_d,
                    h->ctr_d, h->cand_cap);
            h->launches += 1;
        }
        if (!pl.units.empty()) {
            int64_t most = 1;  // counters of the largest owned tile row
            for (const AccUnit& u : pl.units) {
                const Rect& r = pl.rects[u.rect];
                most = std::max<int64_t>(most, (int64_t)std::min(kTile, r.n_rows - u.ti * kTile) * r.n_cols_real);
            }
            const dim3 g((unsigned)std::min<int64_t>((most + 256 * kAccPerThread - 1) / (256 * kAccPerThread), 1024),
                         (unsigned)std::min<size_t>(pl.units.size(), 65535));
            k2_acc_threshold<<<g, 256, 0, st>>>(units_d, (int)pl.units.size(), rects_d, h->cnt_d, sel.f, kp->lw_d,
                                                threshold, use_f, h->cand_d, h->ctr_d, h->cand_cap);
            h->launches += 1;
        }
        cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) {
            set_error("intersection kernel launch: %s", cudaGetErrorString(le));
            rc = BATMAP_E_CUDA;
            break;
        }
        unsigned long long cnt = 0;
        BM_TRY(read_scalar(st, h->ctr_d, &cnt));
        *n_cand = (int64_t)cnt;
        if ((int64_t)cnt <= h->cand_cap) break;
        rc = ensure_cand(h, (int64_t)cnt, st);
        if (rc != BATMAP_OK) break;
    }
    if (kp == &local) release_k2(&local, st);
    return rc;
}

batmap_status swar_device(const uint32_t* x, const uint32_t* y, int64_t n, uint32_t* out, cudaStream_t st) {
    if (n <= 0) return BATMAP_OK;
    k_swar_selftest<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, y, n, out, 1u);
    BM_CUDA(cudaGetLastError());
    return BATMAP_OK;
}

}  // namespace bm
