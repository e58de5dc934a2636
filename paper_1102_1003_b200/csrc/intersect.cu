// intersect.cu -- ★K2: all-pairs BatMap intersection with the fused threshold epilogue.
//
// What is computed: for every selected pair (i, j) with
// W_i <= W_j words,   c_ij = sum_{w < W_j} SWAR(B_j[w], B_i[w mod W_i]),
// SWAR(x, y) = #byte lanes with equal 7 element bits and (b_x OR b_y).
//
// How (B200): the pair triangle is split into width-class rectangles and then
// into 128 x 128 tiles (symmetry cut p <= q).  A persistent CTA per SM walks its
// tiles; one producer warp streams [32 words x 128 items] boxes of both operands with TMA
// (cp.async.bulk.tensor, 4-stage mbarrier ring) -- the narrow operand's box coordinate is
// taken mod W_i, which realises the paper's wrap-around -- and 8 consumer warps compute an
// 8 x 8 register micro-tile of pairs per thread.  Per word pair the SWAR compare-and-count is
// 4 integer instructions (LOP3, IMAD, LOP3, IDP4A: two on the ALU pipe, two on the FMA pipe);
// the indicator masks x&M are derived once per stage into a second shared-memory plane, so
// the ALU pipe (the binding one: half the FMA pipe's rate) sees exactly 2 instructions/compare.  The dot-product accumulates
// 128 x matches in one 32-bit register per pair (exact while 512 W_j < 2^32).  The epilogue
// applies the candidate test c + f_i + f_j >= s (exact corrections follow in finalize.cu) and
// appends candidates with one atomic per warp.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace bm {

constexpr int kBM = 128, kBN = 128, kBK = 32, kConsumerWarps = 8;
constexpr int kThreads = kConsumerWarps * 32;
// K2 variants: BK = words per k-chunk, STAGES = smem ring depth, MINB = CTAs per SM,
// PF = explicit register prefetch of the next k step.
template <int BK>
struct Chunk {
    static constexpr int kStageWords = BK * (kBM + kBN);  // raw words TMA writes per stage
    static constexpr int kStageSmem = 2 * kStageWords;    // + the indicator-mask plane the consumers derive
};
template <int BK, int STAGES>
constexpr size_t smem_bytes() {
    return (size_t)STAGES * Chunk<BK>::kStageSmem * 4 + STAGES * 8;
}
constexpr int kMaxClasses = 26;
constexpr int kMaxTiledW = 1 << 23;  // 512 * W < 2^32 keeps the 128x-scaled counters exact

struct K2Params {
    CUtensorMap maps[kMaxClasses];
    int32_t cls_n[kMaxClasses];
    int32_t cls_W[kMaxClasses];
    int32_t cls_first[kMaxClasses];
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
// (tools/swar_ubench.cu measured this mix at 0.96 of R_int = 32 compares/clk/SM without LDS.)
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

__device__ __forceinline__ void load_ops(Ops& o, const uint32_t* sA, const uint32_t* sB, const uint32_t* mA,
                                         const uint32_t* mB, int k, int tr, int tc) {
    o.xa = *reinterpret_cast<const uint4*>(sA + k * kBM + 4 * tr);
    o.xb = *reinterpret_cast<const uint4*>(sA + k * kBM + 64 + 4 * tr);
    o.ya = *reinterpret_cast<const uint4*>(sB + k * kBN + 4 * tc);
    o.yb = *reinterpret_cast<const uint4*>(sB + k * kBN + 64 + 4 * tc);
    o.ma = *reinterpret_cast<const uint4*>(mA + k * kBM + 4 * tr);
    o.mb = *reinterpret_cast<const uint4*>(mA + k * kBM + 64 + 4 * tr);
    o.na = *reinterpret_cast<const uint4*>(mB + k * kBN + 4 * tc);
    o.nb = *reinterpret_cast<const uint4*>(mB + k * kBN + 64 + 4 * tc);
}

__device__ __forceinline__ void compute_ops(const Ops& o, uint32_t (&acc)[8][8]) {
    const uint32_t x[8] = {o.xa.x, o.xa.y, o.xa.z, o.xa.w, o.xb.x, o.xb.y, o.xb.z, o.xb.w};
    const uint32_t y[8] = {o.ya.x, o.ya.y, o.ya.z, o.ya.w, o.yb.x, o.yb.y, o.yb.z, o.yb.w};
    const uint32_t xm[8] = {o.ma.x, o.ma.y, o.ma.z, o.ma.w, o.mb.x, o.mb.y, o.mb.z, o.mb.w};
    const uint32_t ym[8] = {o.na.x, o.na.y, o.na.z, o.na.w, o.nb.x, o.nb.y, o.nb.z, o.nb.w};
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = swar_step(x[i], y[j], xm[i], ym[j], acc[i][j]);
}

// Per-CTA stream of k-chunks.  Tiles (sorted by cost, longest first) are claimed dynamically
// from a global counter by the CTA's thread 0 -- longest-processing-time order, so the CTAs
// finish within about one (short) tile of each other -- and each tile is split into W_b / BK
// chunks.  The narrow operand's chunk coordinate wraps mod W_a (reading #18).
template <int BK>
struct ChunkCursor {
    int t, kc, nk, ka, Wa;
    int4 td;
    __device__ __forceinline__ bool valid(int n_tiles) const { return t < n_tiles; }
    __device__ __forceinline__ void claim(const K2Params& prm, const int4* tiles, int n_tiles, int* tile_ctr) {
        t = atomicAdd(tile_ctr, 1);
        if (t < n_tiles) {
            td = tiles[t];
            nk = prm.cls_W[td.y] / BK;
            Wa = prm.cls_W[td.x];
            kc = 0;
            ka = 0;
        }
    }
    __device__ __forceinline__ void advance(const K2Params& prm, const int4* tiles, int n_tiles, int* tile_ctr) {
        ++kc;
        ka += BK;
        if (ka == Wa) ka = 0;
        if (kc == nk) claim(prm, tiles, n_tiles, tile_ctr);
    }
};

// Thread 0: fill buffer `buf` with the cursor's next chunk (TMA), or post the end marker once.
template <int BK>
__device__ __forceinline__ void issue_next(const K2Params& prm, ChunkCursor<BK>& c, const int4* tiles, int n_tiles,
                                           int* tile_ctr, uint32_t* stages, int buf, uint64_t* full, int2* meta,
                                           bool& end_sent) {
    if (c.valid(n_tiles)) {
        uint32_t* sA = stages + buf * Chunk<BK>::kStageSmem;
        uint32_t* sB = sA + BK * kBM;
        meta[buf] = make_int2(c.t, c.kc);  // published by the mbarrier's release/acquire
        mbar_expect_tx(&full[buf], Chunk<BK>::kStageWords * 4);
        tma_load_2d(sA, &prm.maps[c.td.x], c.td.z * kBM, c.ka, &full[buf]);  // B_i[w mod W_i]
        tma_load_2d(sB, &prm.maps[c.td.y], c.td.w * kBN, c.kc * BK, &full[buf]);
        c.advance(prm, tiles, n_tiles, tile_ctr);
    } else if (!end_sent) {
        meta[buf] = make_int2(-1, 0);
        mbar_arrive(&full[buf]);
        end_sent = true;
    }
}

// Candidate test c + f_i + f_j >= thr for the thread's 8 x 8 pairs and warp-aggregated append.
__device__ __forceinline__ void tile_epilogue(const K2Params& prm, const int4 td, int tr, int tc, int lane,
                                              const uint32_t (&acc)[8][8], const int32_t* __restrict__ f,
                                              uint32_t thr, uint32_t use_f, Cand* __restrict__ out,
                                              unsigned long long* __restrict__ ctr, int64_t cap) {
    const int a = td.x, b = td.y;
    const int na = prm.cls_n[a], nb = prm.cls_n[b];
    const int fa = prm.cls_first[a], fb = prm.cls_first[b];
    int rows[8], cols[8];
    uint32_t fr[8], fc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        rows[i] = td.z * kBM + (i < 4 ? 4 * tr + i : 64 + 4 * tr + (i - 4));
        cols[i] = td.w * kBN + (i < 4 ? 4 * tc + i : 64 + 4 * tc + (i - 4));
        fr[i] = (use_f && rows[i] < na) ? (uint32_t)__ldg(f + fa + rows[i]) : 0u;
        fc[i] = (use_f && cols[i] < nb) ? (uint32_t)__ldg(f + fb + cols[i]) : 0u;
    }
    uint64_t mask = 0;
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const bool valid = rows[i] < na && cols[j] < nb && (a != b || rows[i] < cols[j]);
            const uint64_t c = acc[i][j] >> 7;
            if (valid && c + fr[i] + fc[j] >= thr) {
                mask |= 1ull << (i * 8 + j);
                ++cnt;
            }
        }
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

// 256 threads = 8 warps; thread (tr, tc) owns rows {4tr..4tr+3, 64+4tr..+3} x cols {4tc.., 64+4tc..}
// of the 128 x 128 tile.  Thread 0 also drives TMA: after the per-chunk barrier every warp has
// finished the previous chunk, so that buffer is refilled with the chunk STAGES-1 ahead.
template <int BK, int STAGES, int MINB, bool PF>
__global__ void __launch_bounds__(kThreads, MINB)
    k2_tiled(const __grid_constant__ K2Params prm, const int4* __restrict__ tiles, int n_tiles, int* tile_ctr,
             const int32_t* __restrict__ f, uint32_t thr, uint32_t use_f, Cand* __restrict__ out,
             unsigned long long* __restrict__ ctr, int64_t cap) {
    extern __shared__ __align__(1024) uint32_t smem_raw[];
    uint32_t* stages = smem_raw;  // keep the shared address space visible to the compiler (LDS, not LD)
    constexpr int kStageWords = Chunk<BK>::kStageWords, kStageSmem = Chunk<BK>::kStageSmem;
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + STAGES * kStageSmem);
    __shared__ int2 meta[STAGES];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    ChunkCursor<BK> pre;  // prefetch cursor (thread 0 only)
    bool end_sent = false;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        pre.claim(prm, tiles, n_tiles, tile_ctr);
        for (int s = 0; s < STAGES - 1; ++s)
            issue_next(prm, pre, tiles, n_tiles, tile_ctr, stages, s, full, meta, end_sent);
    }
    __syncthreads();

    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    int4 td = make_int4(0, 0, 0, 0);
    bool have_tile = false;
    for (uint32_t g = 0;; ++g) {
        const int buf = (int)(g % STAGES);
        mbar_wait(&full[buf], (g / STAGES) & 1u);
        const int2 mt = meta[buf];
        if (mt.y == 0 && have_tile) {  // a new tile (or the end) begins: finish the previous one
            tile_epilogue(prm, td, tr, tc, lane, acc, f, thr, use_f, out, ctr, cap);
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0;
        }
        if (mt.x < 0) break;
        if (mt.y == 0) {
            td = tiles[mt.x];
            have_tile = true;
        }
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
            issue_next(prm, pre, tiles, n_tiles, tile_ctr, stages, (int)((g + STAGES - 1) % STAGES), full, meta,
                       end_sent);
        const uint32_t* sB = sA + BK * kBM;
        const uint32_t* mA = sA + kStageWords;
        const uint32_t* mB = mA + BK * kBM;
        if (PF) {
            Ops cur, nxt;
            load_ops(cur, sA, sB, mA, mB, 0, tr, tc);
#pragma unroll 8
            for (int k = 0; k < BK; ++k) {
                if (k + 1 < BK) load_ops(nxt, sA, sB, mA, mB, k + 1, tr, tc);  // software pipelining
                compute_ops(cur, acc);
                cur = nxt;
            }
        } else {
#pragma unroll 2
            for (int k = 0; k < BK; ++k) {
                Ops cur;
                load_ops(cur, sA, sB, mA, mB, k, tr, tc);
                compute_ops(cur, acc);
            }
        }
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
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
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

// K2 variant (BATMAP_K2_VARIANT=0|1 overrides, for measurement): 0 = one CTA/SM, 32-word chunks,
// register-prefetched operands; 1 = two CTAs/SM (16 warps/SM), 16-word chunks.
static int k2_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("BATMAP_K2_VARIANT");
        v = e ? atoi(e) : 1;
    }
    return v;
}

static batmap_status ensure_cand(batmap_collection* h, int64_t need, cudaStream_t st) {
    return ensure(&h->cand_d, &h->cand_cap, need, st);
}

batmap_status run_intersect(batmap_collection* h, const Selection& sel, uint32_t threshold, int part,
                            int n_parts, uint32_t flags, cudaStream_t st, int64_t* n_cand) {
    *n_cand = 0;
    if (sel.n_sel < 2) return BATMAP_OK;
    bool simple = (flags & BATMAP_PAIRS_SIMPLE) != 0;
    for (const ClassInfo& c : sel.classes)
        if (c.W % 32 != 0 || c.W >= kMaxTiledW) simple = true;
    if ((int)sel.classes.size() > kMaxClasses) simple = true;
    PFN_cuTensorMapEncodeTiled_v12000 enc = simple ? nullptr : tensor_map_encoder();
    if (!simple && !enc) simple = true;

    TileList tl;
    const int tm = simple ? 16 : kBM;
    plan_tiles(sel.classes, tm, part, n_parts, &tl);
    const int64_t n_tiles = (int64_t)tl.tiles.size();
    {  // algorithmic work of this part: sum over its pairs of max(W_i, W_j)
        int64_t wc = 0;
        for (const int4& t : tl.tiles) {
            const ClassInfo &A = sel.classes[t.x], &B = sel.classes[t.y];
            const int64_t rows = std::min<int64_t>(tm, A.n - (int64_t)t.z * tm);
            const int64_t cols = std::min<int64_t>(tm, B.n - (int64_t)t.w * tm);
            const int64_t pairs = (t.x == t.y && t.z == t.w) ? rows * (rows - 1) / 2 : rows * cols;
            wc += pairs * B.W;
        }
        h->stats.word_compares = wc;
        h->stats.tile_compares = tl.work;
        h->stats.k2_kind = simple ? 2 : 1;
        h->stats.k2_grid = simple ? (int32_t)n_tiles
                                  : (int32_t)std::min<int64_t>(n_tiles, (k2_variant() == 0 ? 1 : 2) * h->num_sms);
    }
    if (n_tiles == 0) return BATMAP_OK;
    int4* tiles_d = nullptr;
    BM_TRY(dalloc_t(&tiles_d, n_tiles, st));
    BM_CUDA(cudaMemcpyAsync(tiles_d, tl.tiles.data(), n_tiles * sizeof(int4), cudaMemcpyHostToDevice, st));
    if (!h->ctr_d) BM_TRY(dalloc_t(&h->ctr_d, 2, st));
    if (h->cand_cap == 0) BM_TRY(ensure_cand(h, std::max<int64_t>(1 << 20, sel.n_sel * 16), st));
    const uint32_t use_f = (flags & BATMAP_PAIRS_RAW) ? 0u : 1u;

    SimpleClass* scls_d = nullptr;
    K2Params* prm = nullptr;
    if (simple) {
        std::vector<SimpleClass> sc(sel.classes.size());
        for (size_t a = 0; a < sel.classes.size(); ++a)
            sc[a] = {sel.classes[a].word_off, sel.classes[a].n, sel.classes[a].n_pad, sel.classes[a].W,
                     (int32_t)sel.classes[a].first};
        BM_TRY(dalloc_t(&scls_d, (int64_t)sc.size(), st));
        BM_CUDA(cudaMemcpyAsync(scls_d, sc.data(), sc.size() * sizeof(SimpleClass), cudaMemcpyHostToDevice, st));
        BM_CUDA(cudaStreamSynchronize(st));  // sc is a host temporary
    } else {
        prm = new K2Params();
        for (size_t a = 0; a < sel.classes.size(); ++a) {
            const ClassInfo& c = sel.classes[a];
            cuuint64_t dims[2] = {(cuuint64_t)c.n_pad, (cuuint64_t)c.W};
            cuuint64_t strides[1] = {(cuuint64_t)c.n_pad * 4};
            cuuint32_t box[2] = {(cuuint32_t)kBM, (cuuint32_t)(k2_variant() == 0 ? 32 : 16)};
            cuuint32_t estr[2] = {1, 1};
            CUresult r = enc(&prm->maps[a], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                             const_cast<uint32_t*>(sel.arena + c.word_off), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                delete prm;
                dfree(tiles_d, st);
                set_error("cuTensorMapEncodeTiled failed (%d) for class %zu", (int)r, a);
                return BATMAP_E_CUDA;
            }
            prm->cls_n[a] = c.n;
            prm->cls_W[a] = c.W;
            prm->cls_first[a] = (int32_t)c.first;
        }
        static bool attr_set = false;
        if (!attr_set) {
            BM_CUDA(cudaFuncSetAttribute(k2_tiled<32, 3, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes<32, 3>()));
            BM_CUDA(cudaFuncSetAttribute(k2_tiled<16, 3, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes<16, 3>()));
            attr_set = true;
        }
    }
    batmap_status rc = BATMAP_OK;
    int* tile_ctr = reinterpret_cast<int*>(h->ctr_d + 1);
    for (int attempt = 0; attempt < 2; ++attempt) {
        BM_CUDA(cudaMemsetAsync(h->ctr_d, 0, 2 * sizeof(unsigned long long), st));  // [1] = tile counter
        rec(h, EV_K20, st);
        h->launches += 1;
        if (simple) {
            k2_simple<<<(unsigned)n_tiles, dim3(16, 16), 0, st>>>(sel.arena, scls_d, tiles_d, sel.f, threshold, use_f,
                                                                 h->cand_d, h->ctr_d, h->cand_cap);
        } else if (k2_variant() == 0) {
            const int grid = (int)std::min<int64_t>(n_tiles, h->num_sms);
            k2_tiled<32, 3, 1, true><<<grid, kThreads, smem_bytes<32, 3>(), st>>>(
                *prm, tiles_d, (int)n_tiles, tile_ctr, sel.f, threshold, use_f, h->cand_d, h->ctr_d, h->cand_cap);
        } else {
            const int grid = (int)std::min<int64_t>(n_tiles, 2 * h->num_sms);
            k2_tiled<16, 3, 2, false><<<grid, kThreads, smem_bytes<16, 3>(), st>>>(
                *prm, tiles_d, (int)n_tiles, tile_ctr, sel.f, threshold, use_f, h->cand_d, h->ctr_d, h->cand_cap);
        }
        rec(h, EV_K21, st);
        cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) {
            set_error("intersection kernel launch: %s", cudaGetErrorString(le));
            rc = BATMAP_E_CUDA;
            break;
        }
        unsigned long long cnt = 0;
        BM_CUDA(cudaMemcpyAsync(&cnt, h->ctr_d, sizeof(cnt), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        *n_cand = (int64_t)cnt;
        if ((int64_t)cnt <= h->cand_cap) break;
        rc = ensure_cand(h, (int64_t)cnt, st);
        if (rc != BATMAP_OK) break;
    }
    delete prm;
    dfree(scls_d, st);
    dfree(tiles_d, st);
    return rc;
}

batmap_status swar_device(const uint32_t* x, const uint32_t* y, int64_t n, uint32_t* out, cudaStream_t st) {
    if (n <= 0) return BATMAP_OK;
    k_swar_selftest<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, y, n, out, 1u);
    BM_CUDA(cudaGetLastError());
    return BATMAP_OK;
}

}  // namespace bm
