// triples.cu -- NEXT-4: supports of item TRIPLES with 3-of-4 BatMaps.
//
// The paper leaves itemsets larger than pairs open and sketches this route: store
// every element in d = 3 of d + 1 = 4 tables, so any three sets sharing x all store it in at
// least one common table.  Readings #26-#32 (oracle/batmap3_ref.py follows them
// step by step):
//   #26 four tables, π_1..π_4 from the mixer of reading #3 (keys for t = 0..3);
//   #27 6-bit codes: s3 = min{s : 63·2^s >= m}, ⊥ = code 63; r_i as P:421 with s3; superblocks
//       of 4 r_0: h_t(x) = 4 r_0 floor((π_t(x) mod r)/r_0) + (t-1) r_0 + (π_t(x) mod r_0);
//   #28 INSERT over A_1..A_4 cyclically, called three times per element; failures
//       delete every copy and are corrected exactly (#31);
//   #29 entry = code | B1 << 6 | B2 << 7 (m = the table without x): table 0: B1 = 1; table 1:
//       B1 = [m = 0]; tables 2, 3: B1 = [m = 0], B2 = [m = 1];
//   #30 count at the lowest table common to the three BatMaps: at aligned entries of table t
//       with equal codes, t = 0: B1(a); t = 1: any B1; t = 2: any B1 and any B2; t = 3: any B1,
//       any B2 and any N (m = 2).  Wrap-around as reading #18;
//   #31 supp = c + |{b in S_i ∩ S_j ∩ S_k : b failed in i, j or k}|;
//   #32 candidates = triples whose three pairs are frequent (Apriori property).
//
// Kernels: k3_insert (concurrent INSERT chains, chunks of elements per CTA, uint32 working
// tables in global memory), k3_insert_serial (one thread per item, the reference's order:
// byte-identical), k3_cleanup, k3_encode (element by element, item-major byte arena),
// k3_triples (one warp per candidate, SWAR over the 4 byte lanes of a word), k3_correct,
// k_cand_count / k_cand_emit (Apriori join of the sorted frequent pairs).
#include <algorithm>
#include <type_traits>
#include <cub/cub.cuh>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace bm {

struct Pi4 {
    uint32_t s, w, U, mask, half;
    uint32_t key[4][4];
    const uint32_t* table;  // device [4][U] or nullptr (test hook)
};

__device__ __forceinline__ uint32_t pi4_key(const Pi4& P, int t, int r) {
    return t == 0 ? P.key[0][r] : t == 1 ? P.key[1][r] : t == 2 ? P.key[2][r] : P.key[3][r];
}

__device__ __forceinline__ uint32_t pi4_eval(const Pi4& P, int t, uint32_t x) {
    if (P.table) return __ldg(P.table + (size_t)t * P.U + x);
    uint32_t v = x;
    do {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            v = (v * pi4_key(P, t, r)) & P.mask;
            v ^= v >> P.half;
        }
    } while (v >= P.U);
    return v;
}

// h_t (t 0-based) under the 4-table superblock layout (reading #27)
__device__ __forceinline__ uint32_t slot4(int t, uint32_t v, uint32_t r, uint32_t r0, int log2r0) {
    return 4u * r0 * ((v & (r - 1)) >> log2r0) + (v & (r0 - 1)) + (uint32_t)t * r0;
}

constexpr uint32_t kNull3Word = 0x3F3F3F3Fu;  // four ⊥ entries (reading #27)
constexpr int kChunk3 = 1024;

struct Chunk3 {
    int32_t item, e0, e1, pad;
};

// Concurrent INSERT chains (reading #28 with #9b): each thread inserts its element three times;
// a chain exceeding MaxLoop records its nestless element as failed.  Swaps conserve copies, so
// after all chunks an element with fewer than three copies is exactly a recorded failure.
__global__ void __launch_bounds__(256) k3_insert(const Chunk3* __restrict__ chunks, const int64_t* __restrict__ offsets,
                                                 const int32_t* __restrict__ tids, const int64_t* __restrict__ woff,
                                                 const uint8_t* __restrict__ log2r, Pi4 P, uint32_t r0, int log2r0,
                                                 uint32_t max_loop_opt, uint32_t* __restrict__ work,
                                                 uint64_t* __restrict__ fails, unsigned long long* __restrict__ fail_ctr,
                                                 int64_t fail_cap) {
    const Chunk3 ch = chunks[blockIdx.x];
    const int lr = log2r[ch.item];
    const uint32_t r = 1u << lr;
    const int32_t* S = tids + offsets[ch.item];
    uint32_t* A = work + woff[ch.item];
    const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)lr;
    // persistent lanes: one swap per iteration; a lane whose chain ends (placed, or nestless after
    // MaxLoop rounds) starts its next copy / element at once instead of idling until the warp's
    // longest chain (a failing one runs 4 MaxLoop swaps) ends
    // (one round of the four tables per iteration: the table index stays a compile-time constant,
    // so π's round keys stay kernel-parameter constants)
    int e = ch.e0 + (int)threadIdx.x, copy = 0;
    uint32_t l = 0;
    uint32_t tau = e < ch.e1 ? (uint32_t)__ldg(S + e) : kEmpty;
    while (e < ch.e1) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (tau != kEmpty) tau = atomicExch(&A[slot4(t, pi4_eval(P, t, tau), r, r0, log2r0)], tau);
        if (tau != kEmpty && ++l == max_loop) {  // nestless after MaxLoop rounds: a failure
            const unsigned long long idx = atomicAdd(fail_ctr, 1ull);
            if ((int64_t)idx < fail_cap) fails[idx] = ((uint64_t)ch.item << 32) | tau;
            tau = kEmpty;
        }
        if (tau == kEmpty) {  // chain done: the next copy, or the next element
            l = 0;
            if (++copy == 3) {
                copy = 0;
                e += blockDim.x;
            }
            if (e < ch.e1) tau = (uint32_t)__ldg(S + e);
        }
    }
}

// After concurrent insertion: delete the remaining copies of every element with fewer than three.
__global__ void __launch_bounds__(256) k3_cleanup(const Chunk3* __restrict__ chunks, const int64_t* __restrict__ offsets,
                                                  const int32_t* __restrict__ tids, const int64_t* __restrict__ woff,
                                                  const uint8_t* __restrict__ log2r, Pi4 P, uint32_t r0, int log2r0,
                                                  uint32_t* __restrict__ work) {
    const Chunk3 ch = chunks[blockIdx.x];
    const uint32_t r = 1u << log2r[ch.item];
    const int32_t* S = tids + offsets[ch.item];
    uint32_t* A = work + woff[ch.item];
    for (int e = ch.e0 + threadIdx.x; e < ch.e1; e += blockDim.x) {
        const uint32_t x = (uint32_t)__ldg(S + e);
        uint32_t q[4];
        int cnt = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            q[t] = slot4(t, pi4_eval(P, t, x), r, r0, log2r0);
            cnt += (A[q[t]] == x);
        }
        if (cnt > 0 && cnt < 3)
#pragma unroll
            for (int t = 0; t < 4; ++t) atomicCAS(&A[q[t]], x, kEmpty);
    }
}

// Serial build (BATMAP_BUILD_SERIAL): one thread per item runs INSERT three times per element in
// ascending tid order and the failure cascade of reading #9, exactly as the reference does.
__device__ uint32_t insert4(uint32_t* A, uint32_t tau, const Pi4& P, uint32_t r, uint32_t r0, int log2r0,
                            uint32_t max_loop) {
    for (uint32_t l = 0; l < max_loop; ++l)
        for (int t = 0; t < 4; ++t) {
            const uint32_t q = slot4(t, pi4_eval(P, t, tau), r, r0, log2r0);
            const uint32_t old = A[q];
            A[q] = tau;
            tau = old;
            if (tau == kEmpty) return kEmpty;
        }
    return tau;
}

__global__ void k3_insert_serial(const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids,
                                 const int64_t* __restrict__ woff, const uint8_t* __restrict__ log2r, int64_t n, Pi4 P,
                                 uint32_t r0, int log2r0, uint32_t max_loop_opt, uint32_t* __restrict__ work,
                                 uint64_t* __restrict__ fails, unsigned long long* __restrict__ fail_ctr,
                                 int64_t fail_cap) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int lr = log2r[i];
    const uint32_t r = 1u << lr;
    const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)lr;
    uint32_t* A = work + woff[i];
    for (int64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
        const uint32_t x = (uint32_t)tids[k];
        uint32_t y = kEmpty;
        for (int copy = 0; copy < 3; ++copy) {
            y = insert4(A, x, P, r, r0, log2r0, max_loop);
            if (y != kEmpty) break;
        }
        if (y == kEmpty) continue;
        uint32_t cur = x, nest = y;
        while (true) {
            for (int t = 0; t < 4; ++t) {
                const uint32_t q = slot4(t, pi4_eval(P, t, cur), r, r0, log2r0);
                if (A[q] == cur) A[q] = kEmpty;
            }
            const unsigned long long idx = atomicAdd(fail_ctr, 1ull);
            if ((int64_t)idx < fail_cap) fails[idx] = ((uint64_t)i << 32) | cur;
            if (nest == cur) break;
            const uint32_t z = insert4(A, nest, P, r, r0, log2r0, max_loop);
            if (z == kEmpty) break;
            cur = nest;
            nest = z;
        }
    }
}

// Encode (reading #29), element by element: one CTA per chunk of an item's elements (the chunks of
// k3_insert), one thread per element.  (One warp per item took 1.2 ms on C3: 1,000 warps.)
__global__ void __launch_bounds__(256) k3_encode(const Chunk3* __restrict__ chunks, const int64_t* __restrict__ offsets,
                                                 const int32_t* __restrict__ tids, const int64_t* __restrict__ woff,
                                                 const uint8_t* __restrict__ log2r, Pi4 P, uint32_t r0, int log2r0,
                                                 const uint32_t* __restrict__ work, uint8_t* __restrict__ arena) {
    const Chunk3 ch = chunks[blockIdx.x];
    const uint32_t r = 1u << log2r[ch.item];
    const int32_t* S = tids + offsets[ch.item];
    const uint32_t* A = work + woff[ch.item];
    uint8_t* B = arena + woff[ch.item];  // 4r bytes per item, same offsets as the working table
    for (int e = ch.e0 + threadIdx.x; e < ch.e1; e += blockDim.x) {
        const uint32_t x = (uint32_t)__ldg(S + e);
        uint32_t q[4], cd[4];
        int have = 0, missing = -1;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t v = pi4_eval(P, t, x);
            q[t] = slot4(t, v, r, r0, log2r0);
            cd[t] = v >> P.s;
            if (A[q[t]] == x) ++have;
            else missing = t;
        }
        if (have != 3) continue;  // failed element: no copy left
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (t == missing) continue;
            uint32_t byte = cd[t];
            if (t == 0) byte |= 0x40u;
            else {
                if (missing == 0) byte |= 0x40u;
                if (t >= 2 && missing == 1) byte |= 0x80u;
            }
            B[q[t]] = (uint8_t)byte;
        }
    }
}

// Reading #30 on one word (4 aligned entries of table t) of each of the three BatMaps: the
// number of entries counted.
__device__ __forceinline__ uint32_t triple_word(uint32_t a, uint32_t b, uint32_t c, int t) {
    const uint32_t eab = ~(((a ^ b) | 0xC0C0C0C0u) - 0x01010101u);
    const uint32_t eac = ~(((a ^ c) | 0xC0C0C0C0u) - 0x01010101u);
    uint32_t f = eab & eac;  // bit 6 of each byte: the three codes are equal
    const uint32_t o = a | b | c;
    if (t == 0) f &= a;
    else {
        f &= o;
        if (t >= 2) f &= o >> 1;
        if (t == 3) f &= ~(a | (a >> 1)) | ~(b | (b >> 1)) | ~(c | (c >> 1));
    }
    return __popc(f & 0x40404040u);
}

struct Cand3 {
    uint32_t i, j, k, c;  // positions (width-sorted not needed here: caller ids) and raw count
};

// One warp per candidate triple (caller ids): c = sum over the words of the widest BatMap
// (entries of the narrower ones wrap, reading #18); emit iff c + f_i + f_j + f_k >= threshold.
__global__ void __launch_bounds__(256) k3_triples(const int32_t* __restrict__ cand, int64_t n_cand,
                                                  const int64_t* __restrict__ woff, const uint8_t* __restrict__ log2r,
                                                  const uint8_t* __restrict__ arena, int log2r0,
                                                  const int32_t* __restrict__ f, uint32_t threshold, uint32_t use_f,
                                                  Cand3* __restrict__ out, unsigned long long* __restrict__ ctr,
                                                  int64_t cap) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t qmask = (1u << (log2r0 - 2)) - 1u;  // words per table run: r0 / 4
    for (int64_t z = warp; z < n_cand; z += n_warps) {
        const int32_t it[3] = {cand[3 * z], cand[3 * z + 1], cand[3 * z + 2]};
        const uint32_t* Bw[3];
        uint32_t Wm[3];
        uint32_t W = 0;
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            Bw[u] = reinterpret_cast<const uint32_t*>(arena + woff[it[u]]);
            Wm[u] = (1u << log2r[it[u]]) - 1u;  // words = 4r / 4 = r
            W = max(W, Wm[u] + 1u);
        }
        uint32_t cnt = 0;
        (void)qmask;
        if (log2r0 >= 4 && W % 128 == 0) {  // 4 consecutive words per lane per step: 16-byte loads
            for (uint32_t w = 4 * lane; w < W; w += 128) {
                const uint4 x = __ldg(reinterpret_cast<const uint4*>(Bw[0] + (w & Wm[0])));
                const uint4 y = __ldg(reinterpret_cast<const uint4*>(Bw[1] + (w & Wm[1])));
                const uint4 z = __ldg(reinterpret_cast<const uint4*>(Bw[2] + (w & Wm[2])));
                const int t = (int)((w >> (log2r0 - 2)) & 3u);  // 4 words share a table when r0 >= 16
                cnt += triple_word(x.x, y.x, z.x, t) + triple_word(x.y, y.y, z.y, t) +
                       triple_word(x.z, y.z, z.z, t) + triple_word(x.w, y.w, z.w, t);
            }
        } else {
            for (uint32_t w = lane; w < W; w += 32) {
                const int t = (int)((w >> (log2r0 - 2)) & 3u);  // table of word w (superblocks of r0 words)
                cnt += triple_word(__ldg(Bw[0] + (w & Wm[0])), __ldg(Bw[1] + (w & Wm[1])), __ldg(Bw[2] + (w & Wm[2])),
                                   t);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
        if (lane == 0) {
            const uint32_t slack = use_f ? (uint32_t)(f[it[0]] + f[it[1]] + f[it[2]]) : 0u;
            if (cnt + slack >= threshold) {
                const unsigned long long at = atomicAdd(ctr, 1ull);
                if ((int64_t)at < cap) out[at] = Cand3{(uint32_t)it[0], (uint32_t)it[1], (uint32_t)it[2], cnt};
            }
        }
    }
}

// Grouped variant (r_0 >= 16, so the 4 words of a 16-byte load share a table): one CTA per kG3
// consecutive candidates.  Candidates come sorted by (i, j, k) from the Apriori join, so runs of
// them share (i, j); in a run, B_i's and B_j's words (and the parts of reading #30 that depend on
// them only) are loaded once per 4 words and reused for every k, and only B_k is read per
// candidate: ~1 instead of 3 L2 loads per word-triple on C3 (4.5 candidates per frequent pair).
constexpr int kG3 = 8;
constexpr int kG3Threads = 128;

// Reading #30 with the (a, b) half of a word hoisted out of the loop over k: every value below
// keeps only bit 6 of each byte lane.  With p = ((a ^ c) | 0xC0C0C0C0) - 0x01010101 (bit 6 of ~p:
// the codes of a and c are equal; no borrow crosses a lane) and c1 = c >> 1 (B2 moved to bit 6):
//   t = 0: e0 & a & ~p                   (codes equal, B1 of a)
//   t = 1: e0 & ~p & (o1 | c)            (any B1)
//   t = 2: ... & (o2 | c1)               (and any B2)
//   t = 3: ... & (n | ~(c | c1))         (and some member holding neither)
// and acc += dp4a(f, 0x01010101) adds 64 per counted entry.
struct PairWord {
    uint32_t a, e0, o1, o2, n;
};

template <int T>
__device__ __forceinline__ PairWord pair_word(uint32_t a, uint32_t b) {  // only what table T needs
    constexpr uint32_t M6 = 0x40404040u;
    PairWord p;
    p.a = a;
    p.e0 = ~(((a ^ b) | 0xC0C0C0C0u) - 0x01010101u) & M6;  // codes of a and b equal
    if (T >= 1) p.o1 = (a | b) & M6;
    if (T >= 2) p.o2 = ((a | b) >> 1) & M6;
    if (T == 3) p.n = (~(a | (a >> 1)) | ~(b | (b >> 1))) & M6;
    return p;
}

template <int T>
__device__ __forceinline__ uint32_t triple_word_acc(const PairWord& q, uint32_t c, uint32_t acc) {
    const uint32_t p = ((q.a ^ c) | 0xC0C0C0C0u) - 0x01010101u;
    uint32_t f;
    if (T == 0) {
        f = q.e0 & q.a & ~p;
    } else {
        f = q.e0 & ~p & (q.o1 | c);
        if (T >= 2) {
            const uint32_t c1 = c >> 1;
            f &= q.o2 | c1;
            if (T == 3) f &= q.n | ~(c | c1);
        }
    }
    uint32_t r;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(f), "n"(0x01010101), "r"(acc));
    return r;
}

// One 4-word step for table T.  The B_k words of all kG3 candidates (and the B_i, B_j words of the
// first run) are loaded first, as predicated loads with no branch between them, so a thread keeps
// up to kG3 + 2 L2 requests in flight (one at a time when each load sat behind its candidate's
// branch: ncu showed the kernel latency-bound, long_scoreboard the top stall, ALU pipe 59 %).  Then
// the runs are computed in order; a run after the first loads its B_i, B_j words when it starts.
template <int T>
__device__ __forceinline__ void triples_step(uint32_t w, int nc, const int (&snew)[kG3], const uint32_t (&sW)[kG3],
                                             const int64_t (&soff)[kG3][3], const uint32_t (&swm)[kG3][3],
                                             const uint8_t* __restrict__ arena, uint32_t (&cnt)[kG3]) {
    uint4 cv[kG3];
#pragma unroll
    for (int g = 0; g < kG3; ++g) {
        const bool act = g < nc && w < sW[g];
        const uint4* pc = reinterpret_cast<const uint4*>(arena + soff[g][2]) + ((w & swm[g][2]) >> 2);
        cv[g] = act ? __ldg(pc) : make_uint4(0u, 0u, 0u, 0u);
    }
    // B_i, B_j words of the first run (wrapped, reading #18); every word index is valid after the wrap
    uint4 a = __ldg(reinterpret_cast<const uint4*>(arena + soff[0][0]) + ((w & swm[0][0]) >> 2));
    uint4 b = __ldg(reinterpret_cast<const uint4*>(arena + soff[0][1]) + ((w & swm[0][1]) >> 2));
    PairWord p[4];
    p[0] = pair_word<T>(a.x, b.x);
    p[1] = pair_word<T>(a.y, b.y);
    p[2] = pair_word<T>(a.z, b.z);
    p[3] = pair_word<T>(a.w, b.w);
#pragma unroll
    for (int g = 0; g < kG3; ++g) {
        if (g >= nc) break;
        if (g > 0 && snew[g]) {  // a later run: its own B_i, B_j words
            a = __ldg(reinterpret_cast<const uint4*>(arena + soff[g][0]) + ((w & swm[g][0]) >> 2));
            b = __ldg(reinterpret_cast<const uint4*>(arena + soff[g][1]) + ((w & swm[g][1]) >> 2));
            p[0] = pair_word<T>(a.x, b.x);
            p[1] = pair_word<T>(a.y, b.y);
            p[2] = pair_word<T>(a.z, b.z);
            p[3] = pair_word<T>(a.w, b.w);
        }
        if (w >= sW[g]) continue;
        uint32_t acc = cnt[g];
        acc = triple_word_acc<T>(p[0], cv[g].x, acc);
        acc = triple_word_acc<T>(p[1], cv[g].y, acc);
        acc = triple_word_acc<T>(p[2], cv[g].z, acc);
        cnt[g] = triple_word_acc<T>(p[3], cv[g].w, acc);
    }
}

__global__ void __launch_bounds__(kG3Threads) k3_triples_grouped(const int32_t* __restrict__ cand, int64_t n_cand,
                                                                 const int64_t* __restrict__ woff,
                                                                 const uint8_t* __restrict__ log2r,
                                                                 const uint8_t* __restrict__ arena, int log2r0,
                                                                 const int32_t* __restrict__ f, uint32_t threshold,
                                                                 uint32_t use_f, Cand3* __restrict__ out,
                                                                 unsigned long long* __restrict__ ctr, int64_t cap) {
    __shared__ int32_t sit[kG3][3];
    __shared__ int64_t soff[kG3][3];
    __shared__ uint32_t swm[kG3][3], sW[kG3];
    __shared__ int snew[kG3];
    __shared__ uint32_t sred[kG3][kG3Threads / 32];
    const int64_t z0 = (int64_t)blockIdx.x * kG3;
    const int nc = (int)(n_cand - z0 < kG3 ? n_cand - z0 : kG3);
    if (threadIdx.x < 3 * nc) {
        const int g = threadIdx.x / 3, u = threadIdx.x % 3;
        const int32_t it = cand[3 * z0 + threadIdx.x];
        sit[g][u] = it;
        soff[g][u] = woff[it];
        swm[g][u] = (1u << log2r[it]) - 1u;  // words = 4r / 4 = r
    }
    __syncthreads();
    if (threadIdx.x < nc) {
        const int g = threadIdx.x;
        sW[g] = max(max(swm[g][0], swm[g][1]), swm[g][2]) + 1u;
        snew[g] = g == 0 || sit[g][0] != sit[g - 1][0] || sit[g][1] != sit[g - 1][1];
    }
    __syncthreads();
    uint32_t Wmax = 0;
    for (int g = 0; g < nc; ++g) Wmax = max(Wmax, sW[g]);
    uint32_t cnt[kG3];
#pragma unroll
    for (int g = 0; g < kG3; ++g) cnt[g] = 0;
    for (uint32_t w = 4 * threadIdx.x; w < Wmax; w += 4 * kG3Threads) {
        switch ((w >> (log2r0 - 2)) & 3u) {  // the table of these 4 words (r_0 >= 16)
            case 0: triples_step<0>(w, nc, snew, sW, soff, swm, arena, cnt); break;
            case 1: triples_step<1>(w, nc, snew, sW, soff, swm, arena, cnt); break;
            case 2: triples_step<2>(w, nc, snew, sW, soff, swm, arena, cnt); break;
            default: triples_step<3>(w, nc, snew, sW, soff, swm, arena, cnt); break;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int g = 0; g < kG3; ++g) {
        uint32_t v = cnt[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0) sred[g][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < nc) {
        const int g = threadIdx.x;
        uint32_t c = 0;
#pragma unroll
        for (int q = 0; q < kG3Threads / 32; ++q) c += sred[g][q] >> 6;  // 64 per counted entry
        const uint32_t slack = use_f ? (uint32_t)(f[sit[g][0]] + f[sit[g][1]] + f[sit[g][2]]) : 0u;
        if (c + slack >= threshold) {
            const unsigned long long at = atomicAdd(ctr, 1ull);
            if ((int64_t)at < cap)
                out[at] = Cand3{(uint32_t)sit[g][0], (uint32_t)sit[g][1], (uint32_t)sit[g][2], c};
        }
    }
}

// Variant of the grouped kernel with the CTA's per-candidate parameters hoisted into registers
// before the loop over words (no shared-memory reads and no 64-bit address arithmetic per step), and
// G candidates per CTA (BATMAP_K3_HOIST=4|8 selects it; A/B against k3_triples_grouped).
template <int T, int G>
__device__ __forceinline__ void triples_step_h(uint32_t w, int nc, uint32_t newmask, const uint4* const (&cb)[G],
                                               const uint32_t (&cm)[G], const uint32_t (&cw)[G],
                                               const uint4* const (&ab)[G][2], const uint32_t (&abm)[G][2],
                                               uint32_t (&cnt)[G]) {
    const uint32_t w4 = w >> 2;
    uint4 cv[G];
#pragma unroll
    for (int g = 0; g < G; ++g) cv[g] = w < cw[g] ? __ldg(cb[g] + (w4 & cm[g])) : make_uint4(0u, 0u, 0u, 0u);
    PairWord p[4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        if (g >= nc) break;
        if (g == 0 || (newmask >> g & 1u)) {  // a run starts: its B_i, B_j words (wrapped, reading #18)
            const uint4 a = __ldg(ab[g][0] + (w4 & abm[g][0]));
            const uint4 b = __ldg(ab[g][1] + (w4 & abm[g][1]));
            p[0] = pair_word<T>(a.x, b.x);
            p[1] = pair_word<T>(a.y, b.y);
            p[2] = pair_word<T>(a.z, b.z);
            p[3] = pair_word<T>(a.w, b.w);
        }
        if (w >= cw[g]) continue;
        uint32_t acc = cnt[g];
        acc = triple_word_acc<T>(p[0], cv[g].x, acc);
        acc = triple_word_acc<T>(p[1], cv[g].y, acc);
        acc = triple_word_acc<T>(p[2], cv[g].z, acc);
        cnt[g] = triple_word_acc<T>(p[3], cv[g].w, acc);
    }
}

template <int G>
__global__ void __launch_bounds__(kG3Threads) k3_triples_hoisted(const int32_t* __restrict__ cand, int64_t n_cand,
                                                                 const int64_t* __restrict__ woff,
                                                                 const uint8_t* __restrict__ log2r,
                                                                 const uint8_t* __restrict__ arena, int log2r0,
                                                                 const int32_t* __restrict__ f, uint32_t threshold,
                                                                 uint32_t use_f, Cand3* __restrict__ out,
                                                                 unsigned long long* __restrict__ ctr, int64_t cap) {
    __shared__ int32_t sit[G][3];
    __shared__ int64_t soff[G][3];
    __shared__ uint32_t swm[G][3];
    __shared__ uint32_t sred[G][kG3Threads / 32];
    const int64_t z0 = (int64_t)blockIdx.x * G;
    const int nc = (int)(n_cand - z0 < G ? n_cand - z0 : G);
    if (threadIdx.x < 3 * nc) {
        const int g = threadIdx.x / 3, u = threadIdx.x % 3;
        const int32_t it = cand[3 * z0 + threadIdx.x];
        sit[g][u] = it;
        soff[g][u] = woff[it];
        swm[g][u] = (1u << log2r[it]) - 1u;  // words = 4r / 4 = r
    }
    __syncthreads();
    const uint4* cb[G];
    const uint4* ab[G][2];
    uint32_t cm[G], cw[G], abm[G][2];
    uint32_t newmask = 0, Wmax = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const bool on = g < nc;
        cb[g] = reinterpret_cast<const uint4*>(arena + (on ? soff[g][2] : 0));
        ab[g][0] = reinterpret_cast<const uint4*>(arena + (on ? soff[g][0] : 0));
        ab[g][1] = reinterpret_cast<const uint4*>(arena + (on ? soff[g][1] : 0));
        cm[g] = on ? swm[g][2] >> 2 : 0u;
        abm[g][0] = on ? swm[g][0] >> 2 : 0u;
        abm[g][1] = on ? swm[g][1] >> 2 : 0u;
        cw[g] = on ? max(max(swm[g][0], swm[g][1]), swm[g][2]) + 1u : 0u;
        Wmax = max(Wmax, cw[g]);
        if (on && g > 0 && (sit[g][0] != sit[g - 1][0] || sit[g][1] != sit[g - 1][1])) newmask |= 1u << g;
    }
    uint32_t cnt[G];
#pragma unroll
    for (int g = 0; g < G; ++g) cnt[g] = 0;
    for (uint32_t w = 4 * threadIdx.x; w < Wmax; w += 4 * kG3Threads) {
        switch ((w >> (log2r0 - 2)) & 3u) {  // the table of these 4 words (r_0 >= 16)
            case 0: triples_step_h<0, G>(w, nc, newmask, cb, cm, cw, ab, abm, cnt); break;
            case 1: triples_step_h<1, G>(w, nc, newmask, cb, cm, cw, ab, abm, cnt); break;
            case 2: triples_step_h<2, G>(w, nc, newmask, cb, cm, cw, ab, abm, cnt); break;
            default: triples_step_h<3, G>(w, nc, newmask, cb, cm, cw, ab, abm, cnt); break;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        uint32_t v = cnt[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0) sred[g][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < nc) {
        const int g = threadIdx.x;
        uint32_t c = 0;
#pragma unroll
        for (int q = 0; q < kG3Threads / 32; ++q) c += sred[g][q] >> 6;  // 64 per counted entry
        const uint32_t slack = use_f ? (uint32_t)(f[sit[g][0]] + f[sit[g][1]] + f[sit[g][2]]) : 0u;
        if (c + slack >= threshold) {
            const unsigned long long at = atomicAdd(ctr, 1ull);
            if ((int64_t)at < cap)
                out[at] = Cand3{(uint32_t)sit[g][0], (uint32_t)sit[g][1], (uint32_t)sit[g][2], c};
        }
    }
}

__device__ __forceinline__ bool bsearch_i32(const int32_t* a, int64_t n, int32_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && a[lo] == v;
}

// Exact corrections (reading #31): b counts once if it failed in i, j or k and all three hold b
// (membership in A_b, the sorted items of failed transaction b).  Then re-threshold and emit
// (i, j, k, support) with a 64-bit sort key (i n + j) n + k.  One warp per candidate: the lanes
// share the failures of its three items (dependent binary searches, latency-bound per thread).
__global__ void __launch_bounds__(256) k3_correct(const Cand3* __restrict__ cand, int64_t n_cand,
                                                  const int64_t* __restrict__ fail_off,
                                                  const int32_t* __restrict__ fail_tid,
                                                  const int32_t* __restrict__ fidx_of_tid,
                                                  const int64_t* __restrict__ ab_off, const int32_t* __restrict__ ab_item,
                                                  uint32_t threshold, int64_t n_items, uint64_t* __restrict__ keys,
                                                  uint32_t* __restrict__ vals, unsigned long long* __restrict__ ctr) {
    const int64_t z = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (z >= n_cand) return;  // warp-uniform
    const Cand3 c = cand[z];
    const uint32_t it[3] = {c.i, c.j, c.k};
    uint32_t corr = 0;
    if (fail_off) {
        int64_t f0[3], nf[3];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            f0[u] = fail_off[it[u]];
            nf[u] = fail_off[it[u] + 1] - f0[u];
        }
        for (int64_t q = lane; q < nf[0] + nf[1] + nf[2]; q += 32) {
            const int u = q < nf[0] ? 0 : (q < nf[0] + nf[1] ? 1 : 2);
            const int32_t b = fail_tid[f0[u] + q - (u > 0 ? nf[0] : 0) - (u > 1 ? nf[1] : 0)];
            bool seen = false;  // counted already through an earlier member's failure list
            for (int v = 0; v < u; ++v) seen |= bsearch_i32(fail_tid + f0[v], nf[v], b);
            if (seen) continue;
            const int32_t k = fidx_of_tid[b];
            const int32_t* Ab = ab_item + ab_off[k];
            const int64_t na = ab_off[k + 1] - ab_off[k];
            corr += (bsearch_i32(Ab, na, (int32_t)it[0]) && bsearch_i32(Ab, na, (int32_t)it[1]) &&
                     bsearch_i32(Ab, na, (int32_t)it[2]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) corr += __shfl_xor_sync(0xFFFFFFFFu, corr, o);
    }
    const uint32_t s = c.c + corr;
    if (lane == 0 && s >= threshold) {
        const unsigned long long at = atomicAdd(ctr, 1ull);
        keys[at] = ((uint64_t)c.i * (uint64_t)n_items + c.j) * (uint64_t)n_items + c.k;
        vals[at] = s;
    }
}

__global__ void k3_unpack(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                          int64_t n_items, batmap_quad* __restrict__ out) {
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= n) return;
    const uint64_t key = keys[z];
    const uint64_t k = key % (uint64_t)n_items, ij = key / (uint64_t)n_items;
    out[z] = batmap_quad{(uint32_t)(ij / (uint64_t)n_items), (uint32_t)(ij % (uint64_t)n_items), (uint32_t)k, vals[z]};
}

// ------------------------------------------------------------------ failure bookkeeping
__global__ void k3_mark_failed(const uint64_t* __restrict__ fails, int64_t F, int32_t* __restrict__ mark) {
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (z < F) mark[(uint32_t)fails[z]] = 1;
}

__global__ void k3_fail_split(const uint64_t* __restrict__ fails, int64_t F, int64_t n, int64_t* __restrict__ fail_off,
                              int32_t* __restrict__ fail_tid) {
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (z > F) return;
    const int64_t item = z < F ? (int64_t)(fails[z] >> 32) : n;
    const int64_t prev = z > 0 ? (int64_t)(fails[z - 1] >> 32) : -1;
    for (int64_t q = prev + 1; q <= item; ++q) fail_off[q] = z;
    if (z < F) fail_tid[z] = (int32_t)(uint32_t)fails[z];
}

// one thread per CSR entry: entries whose tid failed somewhere emit key fidx(b) * n + item
__global__ void k3_ab_emit(const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids, int64_t n,
                           int64_t nnz, const int32_t* __restrict__ fidx, uint64_t* __restrict__ keys,
                           unsigned long long* __restrict__ ctr, int64_t cap) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const int32_t f = fidx[tids[k]];
    if (f < 0) return;
    int64_t lo = 0, hi = n - 1;  // the item of entry k
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (offsets[mid] <= k) lo = mid;
        else hi = mid - 1;
    }
    const unsigned long long at = atomicAdd(ctr, 1ull);
    if ((int64_t)at < cap) keys[at] = (uint64_t)f * (uint64_t)n + (uint64_t)lo;
}

__global__ void k3_ab_split(const uint64_t* __restrict__ keys, int64_t total, int64_t n, int64_t nft,
                            int32_t* __restrict__ item, int64_t* __restrict__ off) {
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (z > total) return;
    const int64_t k = z < total ? (int64_t)(keys[z] / (uint64_t)n) : nft;
    const int64_t prev = z > 0 ? (int64_t)(keys[z - 1] / (uint64_t)n) : -1;
    for (int64_t q = prev + 1; q <= k; ++q) off[q] = z;
    if (z < total) item[z] = (int32_t)(keys[z] % (uint64_t)n);
}

__global__ void k3_fail_counts(const int64_t* __restrict__ fail_off, int64_t n, int32_t* __restrict__ f) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) f[i] = (int32_t)(fail_off[i + 1] - fail_off[i]);
}

// fidx[b] holds the exclusive scan of the failed-tid marks: keep it where b failed, -1 elsewhere
__global__ void k3_fidx_final(const int32_t* __restrict__ mark, int64_t m, int32_t* __restrict__ fidx) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < m && !mark[b]) fidx[b] = -1;
}

__global__ void k3_check(const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids, int64_t n, int64_t m,
                         int* __restrict__ bad) {
    const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (item >= n) return;
    const int64_t b = offsets[item], e = offsets[item + 1];
    for (int64_t k = b + lane; k < e; k += 32) {
        const int32_t t = tids[k];
        if (t < 0 || t >= m || (k > b && tids[k - 1] >= t)) atomicOr(bad, 1);
    }
}

__global__ void k3_fill_u32(uint32_t* p, int64_t n, uint32_t v) {
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (z < n) p[z] = v;
}

// ------------------------------------------------------------------ candidates (reading #32)
// rows of the sorted pair list: row_off[i] = first pair with pairs[.].i >= i
__global__ void k_pair_rows(const batmap_triple* __restrict__ pairs, int64_t K, int64_t n, int64_t* __restrict__ row_off) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    int64_t lo = 0, hi = K;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)pairs[mid].i < i) lo = mid + 1;
        else hi = mid;
    }
    row_off[i] = lo;
}

// per pair (i, j): the k > j adjacent to both i and j (two-finger merge of the sorted rows)
template <bool EMIT>
__global__ void k_cand(const batmap_triple* __restrict__ pairs, int64_t K, const int64_t* __restrict__ row_off,
                       const int64_t* __restrict__ at_off, int64_t* __restrict__ count, int32_t* __restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= K) return;
    const uint32_t i = pairs[p].i, j = pairs[p].j;
    int64_t a = p + 1, ae = row_off[i + 1];  // row i after j (rows are sorted by j)
    int64_t b = row_off[j], be = row_off[j + 1];
    int64_t nfound = 0, at = EMIT ? at_off[p] : 0;
    while (a < ae && b < be) {
        const uint32_t x = pairs[a].j, y = pairs[b].j;
        if (x < y) ++a;
        else if (y < x) ++b;
        else {
            if (EMIT) {
                out[3 * at] = (int32_t)i;
                out[3 * at + 1] = (int32_t)j;
                out[3 * at + 2] = (int32_t)x;
                ++at;
            }
            ++nfound;
            ++a;
            ++b;
        }
    }
    if (!EMIT) count[p] = nfound;
}

static inline unsigned gridn(int64_t n, int bs) { return (unsigned)std::max<int64_t>(1, (n + bs - 1) / bs); }

}  // namespace bm

using namespace bm;

// ------------------------------------------------------------------ the 3-of-4 handle
struct batmap3_collection {
    int64_t n = 0, m = 0, nnz = 0;
    int s3 = 0;
    int64_t r0 = 0;
    int log2r0 = 0;
    Pi4 pi{};
    std::vector<uint8_t> lr_h;
    uint8_t* log2r_d = nullptr;
    int64_t* woff_d = nullptr;   // byte offset of item i's 4 r_i bytes (== word offset of its working table)
    uint8_t* arena_d = nullptr;  // item-major 3-of-4 BatMaps
    int64_t arena_bytes = 0;
    int32_t* f_d = nullptr;      // failures per item
    int64_t n_fail = 0, n_ftid = 0;
    int64_t* fail_off_d = nullptr;
    int32_t* fail_tid_d = nullptr;
    int32_t* fidx_d = nullptr;  // m: index of a failed tid or -1
    int64_t* ab_off_d = nullptr;
    int32_t* ab_item_d = nullptr;
    double build_ms = 0, triples_ms = 0;
    int64_t word_triples = 0;
    cudaEvent_t ev[4] = {};
    cudaStream_t stream = nullptr;  // the build's stream: the handle's buffers are allocated on it
};

static void free3(batmap3_collection* h, cudaStream_t st) {
    void* ps[] = {h->log2r_d, h->woff_d, h->arena_d, h->f_d, h->fail_off_d, h->fail_tid_d, h->fidx_d, h->ab_off_d,
                  h->ab_item_d};
    for (void* p : ps) dfree(p, st);  // stream-ordered, into the device pool
    for (cudaEvent_t e : h->ev)
        if (e) cudaEventDestroy(e);
}

// The handle's buffers come from the device pool on the build stream (a plain cudaMalloc of C3's
// 46 MB arena and 184 MB working table took 0.73 ms of host time per build).
template <typename T>
static batmap_status alloc3(batmap3_collection* h, T** p, int64_t count) {
    return dalloc_t(p, count, h->stream);
}

static uint64_t splitmix64_h(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static int ceil_log2(uint64_t v) { return v <= 1 ? 0 : 64 - __builtin_clzll(v - 1); }

// BATMAP_K3_GROUPED=0: the one-warp-per-candidate triple kernel (test hook)
static bool env_flag_off(const char* name) {
    const char* e = getenv(name);
    return e && e[0] == '0';
}

static batmap_status build3(batmap3_collection* h, const int64_t* offsets, const int32_t* tids,
                            const batmap_build_opts* o, cudaStream_t st) {
    const int64_t n = h->n, m = h->m;
    int s3 = 0;
    while ((63ll << s3) < m) ++s3;
    h->s3 = s3;
    Pi4& P = h->pi;
    P.s = (uint32_t)s3;
    P.w = (uint32_t)s3 + 6u;
    P.U = 63u << s3;
    P.mask = P.w >= 32 ? 0xFFFFFFFFu : (1u << P.w) - 1u;
    P.half = (P.w + 1u) / 2u;
    const uint64_t seed = o ? o->seed : 0;
    for (int t = 0; t < 4; ++t)
        for (int r = 0; r < 4; ++r)
            P.key[t][r] = ((uint32_t)splitmix64_h(seed + (uint64_t)(4 * t + r) * 0x9E3779B97F4A7C15ull) | 1u) & P.mask;
    P.table = o ? o->pi_table : nullptr;
    const uint32_t r_min = o && o->r_min ? o->r_min : 128u;
    if (r_min < 4 || (r_min & (r_min - 1))) {
        set_error("r_min must be a power of two >= 4");
        return BATMAP_E_INVALID;
    }
    std::vector<int64_t> off_h(n + 1);
    BM_CUDA(cudaMemcpyAsync(off_h.data(), offsets, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    BM_CUDA(cudaStreamSynchronize(st));
    if (off_h[0] != 0) {
        set_error("offsets[0] must be 0");
        return BATMAP_E_INVALID;
    }
    h->lr_h.resize(n);
    const int lmin = std::max(s3, ceil_log2(r_min));
    std::vector<int64_t> woff(n + 1, 0);
    int lr0 = 62;
    const bool serial = o && (o->flags & BATMAP_BUILD_SERIAL);
    std::vector<Chunk3> chunks;  // items in chunks of elements (k3_insert, k3_cleanup, k3_encode)
    for (int64_t i = 0; i < n; ++i) {
        const int64_t sz = off_h[i + 1] - off_h[i];
        if (sz < 0 || sz > m) {
            set_error("bad offsets at item %lld", (long long)i);
            return BATMAP_E_INVALID;
        }
        const int l = std::max(ceil_log2((uint64_t)(2 * sz)), lmin);
        h->lr_h[i] = (uint8_t)l;
        lr0 = std::min(lr0, l);
        woff[i + 1] = woff[i] + 4ll * (1ll << l);
        for (int64_t e0 = 0; e0 < sz; e0 += kChunk3)
            chunks.push_back({(int32_t)i, (int32_t)e0, (int32_t)std::min<int64_t>(sz, e0 + kChunk3), 0});
    }
    h->nnz = off_h[n];
    h->r0 = n ? (1ll << lr0) : (1ll << lmin);
    h->log2r0 = ceil_log2((uint64_t)h->r0);
    h->arena_bytes = woff[n];
    BM_TRY(alloc3(h, &h->log2r_d, n));
    BM_TRY(alloc3(h, &h->woff_d, n + 1));
    BM_TRY(alloc3(h, &h->arena_d, h->arena_bytes));
    BM_TRY(alloc3(h, &h->f_d, n));
    BM_CUDA(cudaMemcpyAsync(h->log2r_d, h->lr_h.data(), (size_t)n, cudaMemcpyHostToDevice, st));
    BM_CUDA(cudaMemcpyAsync(h->woff_d, woff.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    uint32_t* work = nullptr;
    Chunk3* chunks_d = nullptr;
    uint64_t* fails = nullptr;
    unsigned long long* ctr = nullptr;
    int* bad = nullptr;
    Scratch scratch(st);
    scratch.own(&work);
    scratch.own(&chunks_d);
    scratch.own(&fails);
    scratch.own(&ctr);
    scratch.own(&bad);
    BM_TRY(dalloc_t(&work, h->arena_bytes, st));  // 4 r_i uint32 slots per item (word offsets = byte offsets)
    BM_TRY(dalloc_t(&chunks_d, (int64_t)chunks.size(), st));
    BM_TRY(dalloc_t(&ctr, 2, st));
    if (!chunks.empty())
        BM_CUDA(cudaMemcpyAsync(chunks_d, chunks.data(), chunks.size() * sizeof(Chunk3), cudaMemcpyHostToDevice, st));
    if (o && (o->flags & BATMAP_CHECK_INPUT) && n) {
        BM_TRY(dalloc_t(&bad, 1, st));
        BM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
        // same check as batmap_build: strictly increasing, 0 <= tid < m (one warp per item)
        k3_check<<<gridn(n * 32, 256), 256, 0, st>>>(offsets, tids, n, m, bad);
        int bh = 0;
        BM_TRY(read_scalar(st, bad, &bh));
        if (bh) {
            set_error("invalid tidlists: every tidlist must be strictly increasing in [0, n_transactions)");
            return BATMAP_E_INVALID;
        }
    }
    int64_t fail_cap = std::max<int64_t>(1 << 16, h->nnz / 8), F = 0;
    for (int attempt = 0; attempt < 4; ++attempt) {
        BM_TRY(dalloc_t(&fails, fail_cap, st));
        BM_CUDA(cudaMemsetAsync(work, 0xFF, (size_t)h->arena_bytes * sizeof(uint32_t), st));
        BM_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), st));
        if (serial) {
            k3_insert_serial<<<gridn(n, 32), 32, 0, st>>>(offsets, tids, h->woff_d, h->log2r_d, n, P, (uint32_t)h->r0,
                                                          h->log2r0, o ? o->max_loop : 0u, work, fails, ctr, fail_cap);
        } else if (!chunks.empty()) {
            k3_insert<<<(unsigned)chunks.size(), 256, 0, st>>>(chunks_d, offsets, tids, h->woff_d, h->log2r_d, P,
                                                               (uint32_t)h->r0, h->log2r0, o ? o->max_loop : 0u, work,
                                                               fails, ctr, fail_cap);
            k3_cleanup<<<(unsigned)chunks.size(), 256, 0, st>>>(chunks_d, offsets, tids, h->woff_d, h->log2r_d, P,
                                                                (uint32_t)h->r0, h->log2r0, work);
        }
        BM_CUDA(cudaGetLastError());
        unsigned long long Fh = 0;
        BM_TRY(read_scalar(st, ctr, &Fh));
        F = (int64_t)Fh;
        if (F <= fail_cap) break;
        dfree(fails, st);
        fails = nullptr;
        fail_cap = 2 * F + 1024;
    }
    if (F > fail_cap || !fails) {
        set_error("build3: failure buffer overflow");
        return BATMAP_E_CAPACITY;
    }
    // the byte arena: ⊥ everywhere, then every stored element's three entries
    k3_fill_u32<<<gridn(h->arena_bytes / 4, 256), 256, 0, st>>>(reinterpret_cast<uint32_t*>(h->arena_d),
                                                               h->arena_bytes / 4, kNull3Word);
    if (!chunks.empty())
        k3_encode<<<(unsigned)chunks.size(), 256, 0, st>>>(chunks_d, offsets, tids, h->woff_d, h->log2r_d, P,
                                                           (uint32_t)h->r0, h->log2r0, work, h->arena_d);
    BM_CUDA(cudaGetLastError());
    // F: sort, deduplicate (a concurrent build may record an element once per failed copy), then
    // per-item failure lists Fail(i), f_i, the failed tids and their item lists A_b
    BM_CUDA(cudaMemsetAsync(h->f_d, 0, n * sizeof(int32_t), st));
    h->n_fail = 0;
    h->n_ftid = 0;
    if (F > 0) {
        uint64_t* sorted = nullptr;
        int64_t* nuniq = nullptr;
        void* tmp = nullptr;
        int32_t* mark = nullptr;
        uint64_t* abk = nullptr;
        scratch.own(&sorted);
        scratch.own(&nuniq);
        scratch.own(&tmp);
        scratch.own(&mark);
        scratch.own(&abk);
        BM_TRY(dalloc_t(&sorted, 2 * F, st));
        BM_TRY(dalloc_t(&nuniq, 1, st));
        size_t b1 = 0, b2 = 0, b3 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, b1, fails, sorted, F, 0, 64, st);
        cub::DeviceSelect::Unique(nullptr, b2, sorted, sorted + F, nuniq, F, st);
        cub::DeviceScan::ExclusiveSum(nullptr, b3, mark, mark, m, st);
        BM_TRY(dalloc(&tmp, std::max({b1, b2, b3}), st));
        cub::DeviceRadixSort::SortKeys(tmp, b1, fails, sorted, F, 0, 64, st);
        cub::DeviceSelect::Unique(tmp, b2, sorted, sorted + F, nuniq, F, st);
        int64_t Fu = 0;
        BM_TRY(read_scalar(st, nuniq, &Fu));
        const uint64_t* uf = sorted + F;  // unique (item << 32 | tid), sorted
        F = Fu;
        h->n_fail = F;
        BM_TRY(alloc3(h, &h->fail_off_d, n + 1));
        BM_TRY(alloc3(h, &h->fail_tid_d, F));
        k3_fail_split<<<gridn(F + 1, 256), 256, 0, st>>>(uf, F, n, h->fail_off_d, h->fail_tid_d);
        k3_fail_counts<<<gridn(n, 256), 256, 0, st>>>(h->fail_off_d, n, h->f_d);
        // failed tids: mark, exclusive scan -> index of each failed tid; total = n_ftid
        BM_TRY(dalloc_t(&mark, m + 1, st));
        BM_CUDA(cudaMemsetAsync(mark, 0, (m + 1) * sizeof(int32_t), st));
        k3_mark_failed<<<gridn(F, 256), 256, 0, st>>>(uf, F, mark);
        BM_TRY(alloc3(h, &h->fidx_d, m + 1));
        cub::DeviceScan::ExclusiveSum(tmp, b3, mark, h->fidx_d, m + 1, st);
        int32_t nft = 0;
        BM_TRY(read_scalar(st, h->fidx_d + m, &nft));
        h->n_ftid = nft;
        k3_fidx_final<<<gridn(m, 256), 256, 0, st>>>(mark, m, h->fidx_d);
        // A_b: every CSR entry whose tid failed somewhere -> key fidx * n + item, sorted
        const int64_t cap = std::max<int64_t>(h->n_ftid * 64, 1024);
        int64_t total = 0;
        for (int attempt = 0; attempt < 2; ++attempt) {
            const int64_t c2 = attempt == 0 ? cap : total;
            BM_TRY(dalloc_t(&abk, 2 * c2, st));
            BM_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
            k3_ab_emit<<<gridn(h->nnz, 256), 256, 0, st>>>(offsets, tids, n, h->nnz, h->fidx_d, abk, ctr, c2);
            unsigned long long th = 0;
            BM_TRY(read_scalar(st, ctr, &th));
            total = (int64_t)th;
            if (total <= c2) break;
            dfree(abk, st);
            abk = nullptr;
        }
        size_t b4 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, b4, abk, abk + total, total, 0, 64, st);
        void* tmp2 = nullptr;
        scratch.own(&tmp2);
        BM_TRY(dalloc(&tmp2, b4, st));
        cub::DeviceRadixSort::SortKeys(tmp2, b4, abk, abk + total, total, 0, 64, st);
        BM_TRY(alloc3(h, &h->ab_off_d, h->n_ftid + 1));
        BM_TRY(alloc3(h, &h->ab_item_d, total));
        k3_ab_split<<<gridn(total + 1, 256), 256, 0, st>>>(abk + total, total, n, h->n_ftid, h->ab_item_d, h->ab_off_d);
    }
    BM_CUDA(cudaGetLastError());
    BM_CUDA(cudaStreamSynchronize(st));  // the scratch buffers (stream-ordered) and the CSR are released
    return BATMAP_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

batmap_status batmap3_build(const int64_t* offsets, const int32_t* tids, int64_t n_items, int64_t n_transactions,
                            const batmap_build_opts* opts, batmap_stream_t stream, batmap3_handle* out) {
    if (!out || !offsets || n_items < 0 || n_transactions < 1) {
        set_error("batmap3_build: invalid arguments");
        return BATMAP_E_INVALID;
    }
    *out = nullptr;
    BM_TRY(check_tids_device(offsets, tids, n_items, reinterpret_cast<cudaStream_t>(stream)));
    if (n_transactions >= (1ll << 31) || n_items >= (1ll << 21)) {
        set_error("batmap3_build: n_transactions must be < 2^31 and n_items < 2^21");
        return BATMAP_E_OVERFLOW;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    auto* h = new batmap3_collection();
    h->stream = st;
    h->n = n_items;
    h->m = n_transactions;
    for (cudaEvent_t& e : h->ev) cudaEventCreate(&e);
    cudaEventRecord(h->ev[0], st);
    const batmap_status rc = build3(h, offsets, tids, opts, st);
    if (rc != BATMAP_OK) {
        cudaStreamSynchronize(st);
        free3(h, st);
        delete h;
        return rc;
    }
    cudaEventRecord(h->ev[1], st);
    cudaEventSynchronize(h->ev[1]);
    float ms = 0;
    cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
    h->build_ms = ms;
    *out = h;
    return BATMAP_OK;
}

batmap_status batmap3_triple_supports(batmap3_handle h, const int32_t* triples, int64_t n_triples, uint32_t threshold,
                                      batmap_quad* out, int64_t capacity, int64_t* n_out, batmap_stream_t stream) {
    if (!h || !n_out || n_triples < 0 || (n_triples > 0 && !triples) || (capacity > 0 && !out)) {
        set_error("batmap3_triple_supports: invalid arguments");
        return BATMAP_E_INVALID;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    *n_out = 0;
    if (n_triples == 0) return BATMAP_OK;
    Cand3* cand = nullptr;
    unsigned long long* ctr = nullptr;
    uint64_t* keys = nullptr;
    uint32_t* vals = nullptr;
    void* tmp = nullptr;
    Scratch scratch(st);
    scratch.own(&cand);
    scratch.own(&ctr);
    scratch.own(&keys);
    scratch.own(&vals);
    scratch.own(&tmp);
    BM_TRY(dalloc_t(&ctr, 2, st));
    BM_TRY(dalloc_t(&cand, n_triples, st));
    BM_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), st));
    cudaEventRecord(h->ev[2], st);
    // grouped when the narrowest BatMap has >= 1024 words (C3: r_0 = 2048; measured 2.26 -> 2.09 ms);
    // C1's 256-word BatMaps leave a CTA of 8 candidates one half-occupied step (2.6 -> 4.2 ms)
    const char* ge = getenv("BATMAP_K3_GROUPED");  // 0: never; 1: also below 1024 words (A/B hook)
    const bool grouped = (h->log2r0 >= 10 || (ge && ge[0] == '1' && h->log2r0 >= 4)) && !env_flag_off("BATMAP_K3_GROUPED");
    // candidates per CTA of the hoisted kernel: 4 (measured on C3: 1.56 ms vs 1.81 with 8 and 1.86
    // for the shared-memory-parameter kernel, BATMAP_K3_HOIST=0); 2, 6, 8 are A/B hooks
    const char* he = getenv("BATMAP_K3_HOIST");
    const int hoist = he ? atoi(he) : 4;
    auto launch_h = [&](auto gtag) {
        constexpr int G = decltype(gtag)::value;
        k3_triples_hoisted<G><<<(unsigned)((n_triples + G - 1) / G), kG3Threads, 0, st>>>(
            triples, n_triples, h->woff_d, h->log2r_d, h->arena_d, h->log2r0, h->f_d, threshold, 1u, cand, ctr,
            n_triples);
    };
    if (grouped && hoist == 2) launch_h(std::integral_constant<int, 2>());
    else if (grouped && hoist == 4) launch_h(std::integral_constant<int, 4>());
    else if (grouped && hoist == 6) launch_h(std::integral_constant<int, 6>());
    else if (grouped && hoist == 8) launch_h(std::integral_constant<int, 8>());
    else if (grouped)
        k3_triples_grouped<<<(unsigned)((n_triples + kG3 - 1) / kG3), kG3Threads, 0, st>>>(
            triples, n_triples, h->woff_d, h->log2r_d, h->arena_d, h->log2r0, h->f_d, threshold, 1u, cand, ctr,
            n_triples);
    const unsigned grid = (unsigned)std::min<int64_t>((n_triples + 7) / 8, 148 * 64);
    if (!grouped)
        k3_triples<<<grid, 256, 0, st>>>(triples, n_triples, h->woff_d, h->log2r_d, h->arena_d, h->log2r0, h->f_d,
                                      threshold, 1u, cand, ctr, n_triples);
    BM_CUDA(cudaGetLastError());
    unsigned long long nc = 0;
    BM_TRY(read_scalar(st, ctr, &nc));
    const int64_t NC = (int64_t)nc;
    BM_TRY(dalloc_t(&keys, 2 * std::max<int64_t>(NC, 1), st));
    BM_TRY(dalloc_t(&vals, 2 * std::max<int64_t>(NC, 1), st));
    BM_CUDA(cudaMemsetAsync(ctr + 1, 0, sizeof(unsigned long long), st));
    if (NC)
        k3_correct<<<gridn(NC * 32, 256), 256, 0, st>>>(cand, NC, h->n_fail ? h->fail_off_d : nullptr, h->fail_tid_d,
                                                    h->fidx_d, h->ab_off_d, h->ab_item_d, threshold, h->n, keys, vals,
                                                    ctr + 1);
    unsigned long long K = 0;
    BM_TRY(read_scalar(st, ctr + 1, &K));
    *n_out = (int64_t)K;
    if ((int64_t)K > capacity) {
        set_error("batmap3_triple_supports: %lld results, capacity %lld", (long long)K, (long long)capacity);
        return BATMAP_E_CAPACITY;
    }
    if (K) {
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys + K, vals, vals + K, (int64_t)K, 0, 64, st);
        BM_TRY(dalloc(&tmp, tb, st));
        cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys + K, vals, vals + K, (int64_t)K, 0, 64, st);
        k3_unpack<<<gridn((int64_t)K, 256), 256, 0, st>>>(keys + K, vals + K, (int64_t)K, h->n, out);
    }
    cudaEventRecord(h->ev[3], st);
    BM_CUDA(cudaGetLastError());
    BM_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]);
    h->triples_ms = ms;
    return BATMAP_OK;
}

batmap_status batmap_candidate_triples(const batmap_triple* pairs, int64_t n_pairs, int64_t n_items, int32_t* out,
                                       int64_t capacity, int64_t* n_out, batmap_stream_t stream) {
    if (!n_out || n_pairs < 0 || n_items < 0 || (n_pairs > 0 && !pairs) || (capacity > 0 && !out)) {
        set_error("batmap_candidate_triples: invalid arguments");
        return BATMAP_E_INVALID;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    *n_out = 0;
    if (n_pairs == 0) return BATMAP_OK;
    int64_t* row_off = nullptr;
    int64_t* cnt = nullptr;
    void* tmp = nullptr;
    Scratch scratch(st);
    scratch.own(&row_off);
    scratch.own(&cnt);
    scratch.own(&tmp);
    BM_TRY(dalloc_t(&row_off, n_items + 1, st));
    BM_TRY(dalloc_t(&cnt, n_pairs + 1, st));
    k_pair_rows<<<gridn(n_items + 1, 256), 256, 0, st>>>(pairs, n_pairs, n_items, row_off);
    k_cand<false><<<gridn(n_pairs, 256), 256, 0, st>>>(pairs, n_pairs, row_off, nullptr, cnt, nullptr);
    BM_CUDA(cudaMemsetAsync(cnt + n_pairs, 0, sizeof(int64_t), st));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, cnt, n_pairs + 1, st);
    BM_TRY(dalloc(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, cnt, n_pairs + 1, st);
    int64_t total = 0;
    BM_TRY(read_scalar(st, cnt + n_pairs, &total));
    *n_out = total;
    if (total > capacity) {
        set_error("batmap_candidate_triples: %lld candidates, capacity %lld", (long long)total, (long long)capacity);
        return BATMAP_E_CAPACITY;
    }
    if (total) k_cand<true><<<gridn(n_pairs, 256), 256, 0, st>>>(pairs, n_pairs, row_off, cnt, nullptr, out);
    BM_CUDA(cudaGetLastError());
    BM_CUDA(cudaStreamSynchronize(st));
    return BATMAP_OK;
}

batmap_status batmap3_info(batmap3_handle h, batmap3_info_t* info) {
    if (!h || !info) {
        set_error("batmap3_info: invalid arguments");
        return BATMAP_E_INVALID;
    }
    info->s_shift = h->s3;
    info->r0 = h->r0;
    info->n_items = h->n;
    info->n_transactions = h->m;
    info->arena_bytes = h->arena_bytes;
    info->n_failures = h->n_fail;
    info->n_failed_tids = h->n_ftid;
    info->build_ms = h->build_ms;
    info->triples_ms = h->triples_ms;
    return BATMAP_OK;
}

batmap_status batmap3_export_entries(batmap3_handle h, int32_t item, uint8_t* out, int64_t capacity, int64_t* r_out) {
    if (!h || item < 0 || item >= h->n || !r_out) {
        set_error("batmap3_export_entries: invalid arguments");
        return BATMAP_E_INVALID;
    }
    const int64_t r = 1ll << h->lr_h[item];
    *r_out = r;
    if (capacity < 4 * r || !out) {
        set_error("batmap3_export_entries: capacity %lld < %lld", (long long)capacity, (long long)(4 * r));
        return BATMAP_E_CAPACITY;
    }
    int64_t off = 0;
    for (int32_t i = 0; i < item; ++i) off += 4ll << h->lr_h[i];
    BM_CUDA(cudaMemcpy(out, h->arena_d + off, (size_t)(4 * r), cudaMemcpyDeviceToHost));
    return BATMAP_OK;
}

batmap_status batmap3_export_failures(batmap3_handle h, int32_t* items, int32_t* tids, int64_t capacity,
                                      int64_t* n_out) {
    if (!h || !n_out) {
        set_error("batmap3_export_failures: invalid arguments");
        return BATMAP_E_INVALID;
    }
    *n_out = h->n_fail;
    if (h->n_fail > capacity || (h->n_fail && (!items || !tids))) {
        set_error("batmap3_export_failures: capacity");
        return BATMAP_E_CAPACITY;
    }
    if (!h->n_fail) return BATMAP_OK;
    std::vector<int64_t> off(h->n + 1);
    BM_CUDA(cudaMemcpy(off.data(), h->fail_off_d, (h->n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    BM_CUDA(cudaMemcpy(tids, h->fail_tid_d, h->n_fail * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < h->n; ++i)
        for (int64_t q = off[i]; q < off[i + 1]; ++q) items[q] = (int32_t)i;
    return BATMAP_OK;
}

void batmap3_destroy(batmap3_handle h) {
    if (!h) return;
    cudaDeviceSynchronize();
    free3(h, 0);  // after the device synchronisation: the caller's stream may be gone
    cudaStreamSynchronize(0);
    delete h;
}

}  // extern "C"
