// build.cu -- ★K1: BatMap construction.
//
// Per item (width-sorted position), one thread runs the paper's generalized cuckoo
// INSERT twice per element in ascending tid order (reading #10) on a working
// table of raw tids, handles failures per P:309-310 / reading #9 and records them in F.
// A second kernel encodes each table entry as (b << 7) | (π_t(x) >> s), with
// b from the partner table (Fig. 5, reading #6) and ⊥ = 0x7F (reading #1), and writes the
// words into the class-blocked, word-major arena the intersection kernel reads.
#include <algorithm>
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <cstring>
#include <future>
#include <chrono>
#include <cstdio>

#include "common.cuh"

namespace bm {

// ------------------------------------------------------------------ device: INSERT
__device__ __forceinline__ uint32_t insert_one(uint32_t* A, uint32_t tau, const PiParams& P,
                                               uint32_t r, uint32_t r0, int log2r0,
                                               uint32_t max_loop) {
    for (uint32_t l = 0; l < max_loop; ++l) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            uint32_t q = slot_of(t, pi_eval(P, t, tau), r, r0, log2r0);
            uint32_t old = A[q];
            A[q] = tau;  // τ <-> A_t[h_t(τ)]
            tau = old;
            if (tau == kEmpty) return kEmpty;
        }
    }
    return tau;  // nestless element after MaxLoop rounds
}

__device__ __forceinline__ void delete_all(uint32_t* A, uint32_t x, const PiParams& P, uint32_t r,
                                           uint32_t r0, int log2r0) {
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        uint32_t q = slot_of(t, pi_eval(P, t, x), r, r0, log2r0);
        if (A[q] == x) A[q] = kEmpty;
    }
}

__global__ void __launch_bounds__(128) k1_insert(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids,
    const int32_t* __restrict__ pos2orig, const int64_t* __restrict__ work_off,
    const uint8_t* __restrict__ log2r, int64_t pos_begin, int64_t n, PiParams P, uint32_t r0, int log2r0,
    uint32_t max_loop_opt, uint32_t* __restrict__ work, int32_t* __restrict__ fcount,
    uint64_t* __restrict__ fails, unsigned long long* __restrict__ fail_ctr, int64_t fail_cap) {
    int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= n) return;
    pos += pos_begin;
    const int orig = pos2orig[pos];
    const int64_t b = offsets[orig], e = offsets[orig + 1];
    const int lr = log2r[pos];
    const uint32_t r = 1u << lr;
    const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)lr;
    uint32_t* A = work + work_off[pos - pos_begin];
    int nf = 0;
    for (int64_t k = b; k < e; ++k) {
        const uint32_t x = (uint32_t)__ldg(tids + k);
        uint32_t y = insert_one(A, x, P, r, r0, log2r0, max_loop);  // first copy
        if (y == kEmpty) y = insert_one(A, x, P, r, r0, log2r0, max_loop);  // second copy
        if (y == kEmpty) continue;
        // delete any occurrences of x, re-insert the nestless element unless it is x;
        // a failing re-insertion is handled the same way (reading #9).
        uint32_t cur = x, nest = y;
        while (true) {
            delete_all(A, cur, P, r, r0, log2r0);
            unsigned long long idx = atomicAdd(fail_ctr, 1ull);
            if ((int64_t)idx < fail_cap) fails[idx] = ((uint64_t)pos << 32) | cur;
            ++nf;
            if (nest == cur) break;
            uint32_t z = insert_one(A, nest, P, r, r0, log2r0, max_loop);
            if (z == kEmpty) break;
            cur = nest;
            nest = z;
        }
    }
    fcount[pos] = nf;
}

// ★K1, shared-memory tier (r <= kSmallMaxR): one warp per item.  The 32 lanes evaluate
// π_t and the three slots of every element in parallel; lane 0 then runs the paper's
// sequential INSERT chain (identical order and semantics to k1_insert) on a shared-memory
// table of 16-bit element indices; finally the lanes encode and store the item's words.
constexpr int kSmallMaxR = 8192;
constexpr uint16_t kEmpty16 = 0xFFFF;

__device__ __forceinline__ uint32_t insert_small(uint16_t* A, const uint16_t* slot, int maxS, uint32_t tau,
                                                 uint32_t max_loop) {
    for (uint32_t l = 0; l < max_loop; ++l) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const uint32_t q = slot[t * maxS + tau];
            const uint32_t old = A[q];
            A[q] = (uint16_t)tau;
            tau = old;
            if (tau == kEmpty16) return kEmpty16;
        }
    }
    return tau;
}

__global__ void __launch_bounds__(32) k1_small(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids, const int32_t* __restrict__ pos2orig,
    int64_t first, int W, uint32_t r, int log2r, int maxS, PiParams P, uint32_t r0, int log2r0,
    uint32_t max_loop_opt, uint32_t* __restrict__ arena_cls, int n_pad, int32_t* __restrict__ fcount,
    uint64_t* __restrict__ fails, unsigned long long* __restrict__ fail_ctr, int64_t fail_cap) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint16_t* A = reinterpret_cast<uint16_t*>(sm);              // 3r entries
    uint16_t* slot = A + 3 * r;                                   // [3][maxS]
    uint8_t* code = reinterpret_cast<uint8_t*>(slot + 3 * maxS);  // [3][maxS]
    const int c = blockIdx.x;
    const int lane = threadIdx.x;
    const int64_t pos = first + c;
    const int orig = pos2orig[pos];
    const int64_t b = offsets[orig];
    const int n = (int)(offsets[orig + 1] - b);
    const int32_t* S = tids + b;
    for (uint32_t q = lane; q < 3 * r; q += 32) A[q] = kEmpty16;
    for (int e = lane; e < n; e += 32) {
        const uint32_t x = (uint32_t)__ldg(S + e);
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const uint32_t v = pi_eval(P, t, x);
            slot[t * maxS + e] = (uint16_t)slot_of(t, v, r, r0, log2r0);
            code[t * maxS + e] = (uint8_t)(v >> P.s);
        }
    }
    __syncwarp();
    if (lane == 0) {
        const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)log2r;
        int nf = 0;
        for (int e = 0; e < n; ++e) {  // ascending tid order (reading #10)
            uint32_t y = insert_small(A, slot, maxS, (uint32_t)e, max_loop);
            if (y == kEmpty16) y = insert_small(A, slot, maxS, (uint32_t)e, max_loop);
            if (y == kEmpty16) continue;
            uint32_t cur = (uint32_t)e, nest = y;  // P:310 / reading #9
            while (true) {
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    const uint32_t q = slot[t * maxS + cur];
                    if (A[q] == cur) A[q] = kEmpty16;
                }
                const unsigned long long idx = atomicAdd(fail_ctr, 1ull);
                if ((int64_t)idx < fail_cap) fails[idx] = ((uint64_t)pos << 32) | (uint32_t)S[cur];
                ++nf;
                if (nest == cur) break;
                const uint32_t z = insert_small(A, slot, maxS, nest, max_loop);
                if (z == kEmpty16) break;
                cur = nest;
                nest = z;
            }
        }
        fcount[pos] = nf;
    }
    __syncwarp();
    const uint32_t sb = 3u * r0;
    for (int w = lane; w < W; w += 32) {
        uint32_t word = 0;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const uint32_t q = 4u * (uint32_t)w + l;
            const uint32_t e = A[q];
            uint32_t byte = kNullByte;
            if (e != kEmpty16) {
                const int t = (int)((q % sb) >> log2r0);
                const int t1 = (t + 1) % 3;
                const uint32_t bit = (A[slot[t1 * maxS + e]] == e) ? 0u : 1u;  // Fig. 5
                byte = (bit << 7) | code[t * maxS + e];
            }
            word |= byte << (8 * l);
        }
        arena_cls[(int64_t)w * n_pad + c] = word;
    }
}

// ★K1, concurrent tiers (default).  The paper's INSERT run by many threads of a CTA
// at once on one item's tables: every swap "τ <-> A_t[h_t(τ)]" is an atomic exchange, so each
// table slot holds at most one copy of any element and the number of copies in flight is
// conserved.  A chain that exceeds MaxLoop rounds records its nestless element as failed; after
// all chains end, the remaining copy of every failed element is deleted (P:310 with a
// different attribution of failures, reading #9b) -- the failure set F is exact either way, and
// the corrections of P:469-474 restore every lost occurrence.  The layout depends on thread
// timing; the pair supports do not.  BATMAP_BUILD_SERIAL selects the deterministic
// one-thread-per-item INSERT order instead (byte-identical to oracle/batmap_ref.py).
constexpr int kConcThreads = 128;

// Encode of the concurrent tiers: the thread of element x reads x's three slots, then rewrites
// each slot that holds x as kTagged | byte, byte = (x also in table t+1 ? 0 : 1) << 7 | code
// (Fig. 5).  Only x's thread writes x's slots, and a tagged slot (bit 31 set, low byte the entry)
// never equals an element (element indices and tids are < 2^31), so the reads of the other
// threads are unaffected (reads and rewrites are atomics, so the sanitizer's race check sees no
// plain-access race).  Afterwards every slot is kEmpty (⊥) or tagged.
constexpr uint32_t kTagged = 0x80000000u;
__device__ __forceinline__ uint32_t pack_tagged(uint4 v) {
    const uint32_t e[4] = {v.x, v.y, v.z, v.w};
    uint32_t word = 0;
#pragma unroll
    for (int l = 0; l < 4; ++l) word |= (e[l] == kEmpty ? (uint32_t)kNullByte : (e[l] & 0xFFu)) << (8 * l);
    return word;
}
constexpr int kConcFailCap = 512;  // per-item failure list in shared memory (overflow -> global rescan)

__device__ __forceinline__ void record_failure(uint32_t* fl, int* nfl, uint64_t* fails, unsigned long long* fail_ctr,
                                               int64_t fail_cap, int64_t pos, uint32_t tid_val, uint32_t e,
                                               int* overflow) {
    const int k = atomicAdd(nfl, 1);
    if (k < kConcFailCap) fl[k] = e;
    else *overflow = 1;
    const unsigned long long idx = atomicAdd(fail_ctr, 1ull);
    if ((int64_t)idx < fail_cap) fails[idx] = ((uint64_t)pos << 32) | tid_val;
}

__global__ void __launch_bounds__(kConcThreads) k1_conc_small(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids, const int32_t* __restrict__ pos2orig,
    int64_t first, int W, uint32_t r, int log2r, int maxS, PiParams P, uint32_t r0, int log2r0,
    uint32_t max_loop_opt, uint32_t* __restrict__ arena_cls, int n_pad, int32_t* __restrict__ fcount,
    uint64_t* __restrict__ fails, unsigned long long* __restrict__ fail_ctr, int64_t fail_cap) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint32_t* A = reinterpret_cast<uint32_t*>(sm);                   // 3r entries (element index)
    uint16_t* slot = reinterpret_cast<uint16_t*>(A + 3 * r);          // [3][maxS]
    uint8_t* code = reinterpret_cast<uint8_t*>(slot + 3 * maxS);      // [3][maxS]
    __shared__ uint32_t fl[kConcFailCap];
    __shared__ int nfl, overflow;
    const int c = blockIdx.x;
    const int64_t pos = first + c;
    const int orig = pos2orig[pos];
    const int64_t b = offsets[orig];
    const int n = (int)(offsets[orig + 1] - b);
    const int32_t* S = tids + b;
    if (threadIdx.x == 0) {
        nfl = 0;
        overflow = 0;
    }
    for (uint32_t q = threadIdx.x; q < 3 * r; q += blockDim.x) A[q] = kEmpty;
    // four tids per thread loaded ahead of the π evaluations (the loads are independent)
    for (int e0 = threadIdx.x; e0 < n; e0 += 4 * blockDim.x) {
        uint32_t xs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * blockDim.x;
            xs[u] = e < n ? (uint32_t)__ldg(S + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e >= n) break;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const uint32_t v = pi_eval(P, t, xs[u]);
                slot[t * maxS + e] = (uint16_t)slot_of(t, v, r, r0, log2r0);
                code[t * maxS + e] = (uint8_t)(v >> P.s);
            }
        }
    }
    __syncthreads();
    const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)log2r;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        for (int copy = 0; copy < 2; ++copy) {  // the insert procedure is called twice
            uint32_t tau = (uint32_t)e;
            for (uint32_t l = 0; l < max_loop && tau != kEmpty; ++l)
#pragma unroll
                for (int t = 0; t < 3 && tau != kEmpty; ++t) tau = atomicExch(&A[slot[t * maxS + tau]], tau);
            if (tau != kEmpty)
                record_failure(fl, &nfl, fails, fail_ctr, fail_cap, pos, (uint32_t)S[tau], tau, &overflow);
        }
    }
    __syncthreads();
    // delete every remaining copy of a failed element
    const int nf = nfl;
    if (!overflow) {
        for (int k = threadIdx.x; k < nf; k += blockDim.x) {
            const uint32_t e = fl[k];
#pragma unroll
            for (int t = 0; t < 3; ++t) atomicCAS(&A[slot[t * maxS + e]], e, kEmpty);
        }
    } else {  // rare: many failures -- any element with fewer than two copies was recorded
        for (int e = threadIdx.x; e < n; e += blockDim.x) {
            int cnt = 0;
#pragma unroll
            for (int t = 0; t < 3; ++t) cnt += (A[slot[t * maxS + e]] == (uint32_t)e);
            if (cnt == 1)
#pragma unroll
                for (int t = 0; t < 3; ++t) atomicCAS(&A[slot[t * maxS + e]], (uint32_t)e, kEmpty);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) fcount[pos] = nf;
    // encode (Fig. 5) element by element, then pack
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        uint32_t q[3];
        bool in[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            q[t] = slot[t * maxS + e];
            in[t] = atomicOr(&A[q[t]], 0u) == (uint32_t)e;  // atomic: other threads tag their slots
        }
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if (in[t]) atomicExch(&A[q[t]], kTagged | (in[(t + 1) % 3] ? 0u : 0x80u) | code[t * maxS + e]);
    }
    __syncthreads();
    for (int w = threadIdx.x; w < W; w += blockDim.x)
        arena_cls[(int64_t)w * n_pad + c] = pack_tagged(reinterpret_cast<const uint4*>(A)[w]);
}

// Concurrent tier for medium tables (kSmallMaxR < r <= kClusterMaxR): one thread-block cluster
// per item; the item's 3r-entry working table (raw tids) is spread over the distributed shared
// memory of the cluster's CS CTAs (slice q / (3r/CS) of slot q), so every swap of the paper's
// INSERT is an on-chip atomic exchange, local or remote (DSMEM).  Same protocol as
// k1_conc_small (reading #9b); π is recomputed on every swap.  The encode (Fig. 5)
// follows in the same kernel, each CTA encoding the words of its own slice.
constexpr uint32_t kClusterMaxR = 131072;
constexpr int kClSliceBytesMax = 3 * 16384 * 4;  // 192 KB of table per CTA

// DSMEM access: slot q of the item's table as (owning CTA, offset); local slots use plain shared
// atomics, remote ones the shared::cluster window (mapa + atom/ld.shared::cluster)
__device__ __forceinline__ uint32_t cl_exch(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t cl_cas(uint32_t addr, uint32_t cmp, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(addr), "r"(cmp), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t cl_ld(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t cl_or0(uint32_t addr) {
    uint32_t old;
    asm volatile("atom.shared::cluster.or.b32 %0, [%1], 0;" : "=r"(old) : "r"(addr) : "memory");
    return old;
}

template <int CS, int NT>
__global__ void __launch_bounds__(NT) k1_conc_cluster(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids, const int32_t* __restrict__ pos2orig,
    int64_t first, uint32_t r, int log2r, PiParams P, uint32_t r0, int log2r0, uint32_t max_loop_opt,
    uint32_t* __restrict__ arena_cls, int n_pad, uint64_t* __restrict__ fails, unsigned long long* __restrict__ fail_ctr,
    int64_t fail_cap, uint32_t* __restrict__ stage) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) uint32_t T[];  // this CTA's slice: 3r / CS entries
    __shared__ uint32_t fl[kConcFailCap];
    __shared__ int nfl, overflow;
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t rank = CS == 1 ? 0u : cl.block_rank();
    const uint32_t slice = 3u * r / CS;
    const int c = blockIdx.x / CS;
    const int64_t pos = first + c;
    const int orig = pos2orig[pos];
    const int64_t b = offsets[orig];
    const int n = (int)(offsets[orig + 1] - b);
    const int32_t* S = tids + b;
    const uint32_t T_loc = (uint32_t)__cvta_generic_to_shared(T);  // CTA k's copy is a mapa away
    // slot q lives in CTA k = floor(q * CS / (3 * 2^log2r)) at offset q - k * slice
    auto owner = [&](uint32_t q) -> uint32_t { return CS == 1 ? 0u : ((q * CS) >> log2r) / 3u; };
    auto exch = [&](uint32_t q, uint32_t v) -> uint32_t {
        const uint32_t k = owner(q), off = q - k * slice;
        if (CS == 1 || k == rank) return atomicExch(T + off, v);
        uint32_t a;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(T_loc + 4u * off), "r"(k));
        return cl_exch(a, v);
    };
    auto cas = [&](uint32_t q, uint32_t cmp, uint32_t v) -> uint32_t {
        const uint32_t k = owner(q), off = q - k * slice;
        if (CS == 1 || k == rank) return atomicCAS(T + off, cmp, v);
        uint32_t a;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(T_loc + 4u * off), "r"(k));
        return cl_cas(a, cmp, v);
    };
    auto load = [&](uint32_t q) -> uint32_t {
        const uint32_t k = owner(q), off = q - k * slice;
        if (CS == 1 || k == rank) return T[off];
        uint32_t a;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(T_loc + 4u * off), "r"(k));
        return cl_ld(a);
    };
    auto read = [&](uint32_t q) -> uint32_t {  // atomic read (the encode runs beside other threads' tagging)
        const uint32_t k = owner(q), off = q - k * slice;
        if (CS == 1 || k == rank) return atomicOr(T + off, 0u);
        uint32_t a;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(T_loc + 4u * off), "r"(k));
        return cl_or0(a);
    };
    for (uint32_t q = threadIdx.x; q < slice; q += NT) T[q] = kEmpty;
    if (threadIdx.x == 0) {
        nfl = 0;
        overflow = 0;
    }
    if (CS > 1) cl.sync();
    else __syncthreads();
    const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)log2r;
    for (int e = (int)rank * NT + threadIdx.x; e < n; e += CS * NT) {
        const uint32_t x = (uint32_t)__ldg(S + e);
        for (int copy = 0; copy < 2; ++copy) {  // the insert procedure is called twice
            uint32_t tau = x;
            for (uint32_t l = 0; l < max_loop && tau != kEmpty; ++l)
#pragma unroll
                for (int t = 0; t < 3 && tau != kEmpty; ++t) tau = exch(slot_of(t, pi_eval(P, t, tau), r, r0, log2r0), tau);
            if (tau != kEmpty) record_failure(fl, &nfl, fails, fail_ctr, fail_cap, pos, tau, tau, &overflow);
        }
    }
    __syncthreads();
    int any_overflow;
    if (CS > 1) {
        int* ovf0 = cl.map_shared_rank(&overflow, 0);
        if (threadIdx.x == 0 && overflow && rank != 0) atomicOr(ovf0, 1);
        cl.sync();
        any_overflow = *ovf0;
    } else {
        any_overflow = overflow;
    }
    if (!any_overflow) {  // delete the remaining copy of every failed element (reading #9b)
        const int nf = nfl;
        for (int k = threadIdx.x; k < nf; k += NT) {
            const uint32_t x = fl[k];
#pragma unroll
            for (int t = 0; t < 3; ++t) cas(slot_of(t, pi_eval(P, t, x), r, r0, log2r0), x, kEmpty);
        }
    } else {  // rare: any element left with fewer than two copies was recorded
        for (int e = (int)rank * NT + threadIdx.x; e < n; e += CS * NT) {
            const uint32_t x = (uint32_t)S[e];
            uint32_t q[3];
            int cnt = 0;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                q[t] = slot_of(t, pi_eval(P, t, x), r, r0, log2r0);
                cnt += (load(q[t]) == x);
            }
            if (cnt == 1)
#pragma unroll
                for (int t = 0; t < 3; ++t) cas(q[t], x, kEmpty);
        }
    }
    if (CS > 1) cl.sync();
    else __syncthreads();
    // encode (Fig. 5) element by element, then every CTA packs the words of its slice
    for (int e = (int)rank * NT + threadIdx.x; e < n; e += CS * NT) {
        const uint32_t x = (uint32_t)__ldg(S + e);
        uint32_t q[3], code[3];
        bool in[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const uint32_t v = pi_eval(P, t, x);
            q[t] = slot_of(t, v, r, r0, log2r0);
            code[t] = v >> P.s;
            in[t] = read(q[t]) == x;
        }
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if (in[t]) exch(q[t], kTagged | (in[(t + 1) % 3] ? 0u : 0x80u) | code[t]);
    }
    if (CS > 1) cl.sync();
    else __syncthreads();
    const uint32_t q0 = rank * slice;
    if (CS == 1 && stage) {  // the item's words as one contiguous row of the staging block (coalesced;
                             // k_pack_transpose writes the arena), as the byte tier does
        for (uint32_t wl = threadIdx.x; wl < slice / 4; wl += NT)
            stage[(int64_t)c * (slice / 4) + wl] = pack_tagged(reinterpret_cast<const uint4*>(T)[wl]);
    } else {
        for (uint32_t wl = threadIdx.x; wl < slice / 4; wl += NT)
            arena_cls[(int64_t)(q0 / 4 + wl) * n_pad + c] = pack_tagged(reinterpret_cast<const uint4*>(T)[wl]);
    }
    if (CS > 1) cl.sync();  // no CTA may exit while another still reads its slice
}


// ------------------------------------------------------------------ byte-table tier
// The working table of an item holds the entry bytes themselves (3r bytes instead of 12r): slot q of
// table t holds code = π_t(x) >> s of the element x placed there, ⊥ = 0x7F (reading #1).
// Slot and code determine v = π_t(x) (r >= 2^s: the slot gives v mod r, the code v >> s), so an
// element evicted by a swap is recovered as x = π_t^-1(v) and continues into table t+1.
// A table of up to r = 2^16 (192 KB) fits ONE CTA's shared memory, so every swap is a local
// shared-memory atomic: the uint32 tier needs a cluster of 4 CTAs and remote DSMEM atomics for the
// same item.  A swap is a byte exchange done as a 32-bit CAS on the word holding the byte (no 8-bit
// exchange exists).  Larger tables (r <= 2^19) spread over a cluster of CS CTAs as before.
// The second INSERT of x starts with τ <-> A_1[h_1(x)]; when that slot still holds x this swap
// exchanges x with itself, so a read replaces it (an atomic fewer per element, same semantics).
// Encode (Fig. 5): the thread of x reads x's three bytes and sets b = 1 with a plain byte
// store on the copy whose partner sits in the preceding table -- x's bytes are written by x's thread
// only, so no atomics are needed -- and the pack pass copies the table words to the arena unchanged.
constexpr uint32_t kByteSliceMax = 3u * 65536u;  // 192 KB of table bytes per CTA
constexpr uint32_t kByteMaxR = 1u << 19;          // CS = 8 x 192 KB

__device__ __forceinline__ uint32_t sh_ld_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t sh_cas(uint32_t a, uint32_t cmp, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t sh_ld_u8(uint32_t a) {
    uint16_t v;
    asm volatile("ld.volatile.shared.u8 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t cl_ld_u8(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared::cluster.u8 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sh_st_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"((uint16_t)v) : "memory");
}
__device__ __forceinline__ void cl_st_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(a), "h"((uint16_t)v) : "memory");
}

// One CTA (CS = 1) builds IPC consecutive items of a class, each in its own 3r-byte slice (padded
// by 16 bytes so the pack's lanes hit distinct banks), or one item is spread over a cluster of CS
// CTAs (IPC = 1).  The INSERT chains run as persistent lanes: a lane whose chain ends takes its next
// task (the element's second INSERT, or the next element) at once instead of idling until the
// warp's slowest chain is done; π's round keys of the table a lane is at come from shared memory.
// The pack writes word w of the IPC items as IPC consecutive arena columns: whole 32-byte sectors
// when IPC = 8.
template <int CS, int IPC, int NT>
__global__ void __launch_bounds__(NT) k1_byte(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids, const int32_t* __restrict__ pos2orig,
    int64_t first, int n_cls, uint32_t r, int log2r, PiParams P, uint32_t r0, int log2r0, uint32_t max_loop_opt,
    uint32_t* __restrict__ arena_cls, int n_pad, uint64_t* __restrict__ fails, unsigned long long* __restrict__ fail_ctr,
    int64_t fail_cap, uint32_t* __restrict__ stage) {
    static_assert(CS == 1 || IPC == 1, "an item spread over a cluster is built alone");
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) uint8_t TB[];  // IPC item slices (CS = 1) or this CTA's slice of one item
    __shared__ uint32_t fl[kConcFailCap];
    __shared__ uint8_t fl_k[kConcFailCap];
    __shared__ int nfl, overflow;
    __shared__ int pre[IPC + 1];
    __shared__ const int32_t* Sk[IPC];
    __shared__ __align__(16) uint32_t keys[3][8];  // per table: 4 forward, 4 inverse round keys
    const uint32_t rank = CS == 1 ? 0u : cg::this_cluster().block_rank();
    const uint32_t slice = 3u * r / CS;
    const uint32_t stride_b = IPC == 1 ? slice : slice + 16u;  // item k's slice at TB + k * stride_b
    const int c0 = (int)(blockIdx.x / CS) * IPC;                // first column of this CTA (cluster)
    const int n_it = max(0, min(IPC, n_cls - c0));
    if (threadIdx.x <= IPC) {
        int cnt = 0;
        for (int k = 0; k < (int)threadIdx.x && k < n_it; ++k) {
            const int orig = pos2orig[first + c0 + k];
            cnt += (int)(offsets[orig + 1] - offsets[orig]);
        }
        pre[threadIdx.x] = cnt;
        if ((int)threadIdx.x < n_it) Sk[threadIdx.x] = tids + offsets[pos2orig[first + c0 + threadIdx.x]];
    }
    if (threadIdx.x == 32) {  // compile-time indices: the parameter struct stays in constant space
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                keys[t][j] = pi_key(P, t, j);
                keys[t][4 + j] = pi_kinv(P, t, j);
            }
    }
    const uint32_t T_loc = (uint32_t)__cvta_generic_to_shared(TB);
    const uint32_t low_s = (1u << P.s) - 1u;
    // slot q of item k -> shared-window address of its byte (remote for another CTA of the cluster)
    auto where = [&](int k, uint32_t q, bool* local) -> uint32_t {
        if (CS == 1) {
            *local = true;
            return T_loc + (uint32_t)k * stride_b + q;
        }
        const uint32_t o = ((q * CS) >> log2r) / 3u;
        const uint32_t a = T_loc + (q - o * slice);
        *local = o == rank;
        if (*local) return a;
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(o));
        return ra;
    };
    auto read_byte = [&](int k, uint32_t q) -> uint32_t {
        bool loc;
        const uint32_t a = where(k, q, &loc);
        return loc ? sh_ld_u8(a) : cl_ld_u8(a);
    };
    // byte exchange (τ <-> A_t[h_t(τ)]): CAS on the word holding the byte; returns the old byte
    auto xchg = [&](int k, uint32_t q, uint32_t code) -> uint32_t {
        bool loc;
        const uint32_t a = where(k, q, &loc);
        const uint32_t wa = a & ~3u, sh = (a & 3u) * 8u;
        uint32_t old = loc ? sh_ld_u32(wa) : cl_ld(wa);
        while (true) {
            const uint32_t nw = (old & ~(0xFFu << sh)) | (code << sh);
            const uint32_t prev = loc ? sh_cas(wa, old, nw) : cl_cas(wa, old, nw);
            if (prev == old) return (old >> sh) & 0xFFu;
            old = prev;
        }
    };
    // byte -> ⊥ if it still holds `code` (deleting a failed element's remaining copy)
    auto erase = [&](int k, uint32_t q, uint32_t code) {
        bool loc;
        const uint32_t a = where(k, q, &loc);
        const uint32_t wa = a & ~3u, sh = (a & 3u) * 8u;
        uint32_t old = loc ? sh_ld_u32(wa) : cl_ld(wa);
        while (((old >> sh) & 0xFFu) == code) {
            const uint32_t nw = (old & ~(0xFFu << sh)) | (kNullByte << sh);
            const uint32_t prev = loc ? sh_cas(wa, old, nw) : cl_cas(wa, old, nw);
            if (prev == old) return;
            old = prev;
        }
    };
    for (uint32_t i = threadIdx.x; i < (uint32_t)IPC * stride_b / 16; i += NT)
        reinterpret_cast<uint4*>(TB)[i] = make_uint4(kNullWord, kNullWord, kNullWord, kNullWord);
    if (threadIdx.x == 0) {
        nfl = 0;
        overflow = 0;
    }
    if (CS > 1) cg::this_cluster().sync();
    else __syncthreads();
    const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)log2r;
    const int ntot = pre[n_it];
    // π_t with table t's round keys from shared memory (t differs between lanes); walk as pi_eval
    auto pi_fwd = [&](int t, uint32_t v) -> uint32_t {
        const uint4 kf = *reinterpret_cast<const uint4*>(&keys[t][0]);
        do {
            v = (v * kf.x) & P.mask;
            v ^= v >> P.half;
            v = (v * kf.y) & P.mask;
            v ^= v >> P.half;
            v = (v * kf.z) & P.mask;
            v ^= v >> P.half;
            v = (v * kf.w) & P.mask;
            v ^= v >> P.half;
        } while (v >= P.U);
        return v;
    };
    auto pi_inv = [&](int t, uint32_t v) -> uint32_t {
        const uint4 ki = *reinterpret_cast<const uint4*>(&keys[t][4]);
        do {
            v ^= v >> P.half;
            v = (v * ki.w) & P.mask;
            v ^= v >> P.half;
            v = (v * ki.z) & P.mask;
            v ^= v >> P.half;
            v = (v * ki.y) & P.mask;
            v ^= v >> P.half;
            v = (v * ki.x) & P.mask;
        } while (v >= P.U);
        return v;
    };
    // ---- INSERT chains as persistent lanes (reading #9b)
    {
        int g = (int)rank * NT + threadIdx.x;  // next element of this lane (flattened over the IPC items)
        int k = 0, t = 0, copy = 0;
        uint32_t x = 0, tau = 0, rounds = 0;
        bool have = false;
        auto begin_element = [&]() {
            have = g < ntot;
            if (!have) return;
            k = 0;
#pragma unroll
            for (int j = 1; j < IPC; ++j) k += (g >= pre[j]);
            x = (uint32_t)__ldg(Sk[k] + (g - pre[k]));
            tau = x;
            t = 0;
            rounds = 0;
            copy = 0;
        };
        begin_element();
        while (__any_sync(0xFFFFFFFFu, have)) {
            if (!have) continue;
            const uint32_t v = pi_fwd(t, tau);
            const uint32_t q = slot_of(t, v, r, r0, log2r0);
            const uint32_t old = xchg(k, q, v >> P.s);
            bool end = old == kNullByte;
            if (!end) {  // the evicted element: v' = π_t(y) from slot and code
                const uint32_t vr = (((q >> log2r0) / 3u) << log2r0) | (q & (r0 - 1u));
                tau = pi_inv(t, (old << P.s) | (vr & low_s));
                if (++t == 3) {
                    t = 0;
                    if (++rounds == max_loop) {  // nestless after MaxLoop rounds: a failure
                        const int j = atomicAdd(&nfl, 1);
                        if (j < kConcFailCap) {
                            fl[j] = tau;
                            fl_k[j] = (uint8_t)k;
                        } else {
                            overflow = 1;
                        }
                        const unsigned long long idx = atomicAdd(fail_ctr, 1ull);
                        if ((int64_t)idx < fail_cap) fails[idx] = ((uint64_t)(first + c0 + k) << 32) | tau;
                        end = true;
                    }
                }
            }
            if (end) {
                if (copy == 0) {  // the insert procedure is called twice
                    copy = 1;
                    tau = x;
                    rounds = 0;
                    // its first swap, τ <-> A_1[h_1(x)], would return x itself if x still sits there
                    const uint32_t v1 = pi_fwd(0, x);
                    t = read_byte(k, slot_of(0, v1, r, r0, log2r0)) == (v1 >> P.s) ? 1 : 0;
                } else {
                    g += CS * NT;
                    begin_element();
                }
            }
        }
    }
    __syncthreads();
    int any_overflow;
    if (CS > 1) {
        cg::cluster_group cl = cg::this_cluster();
        int* ovf0 = cl.map_shared_rank(&overflow, 0);
        if (threadIdx.x == 0 && overflow && rank != 0) atomicOr(ovf0, 1);
        cl.sync();
        any_overflow = *ovf0;
    } else {
        any_overflow = overflow;
    }
    if (!any_overflow) {  // delete the remaining copy of every failed element (reading #9b)
        const int nf = nfl;
        for (int j = threadIdx.x; j < nf; j += NT) {
            const uint32_t x = fl[j];
            const int k = fl_k[j];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const uint32_t v = pi_fwd(t, x);
                erase(k, slot_of(t, v, r, r0, log2r0), v >> P.s);
            }
        }
    } else {  // rare: any element left with fewer than two copies was recorded
        for (int g = (int)rank * NT + threadIdx.x; g < ntot; g += CS * NT) {
            int k = 0;
#pragma unroll
            for (int j = 1; j < IPC; ++j) k += (g >= pre[j]);
            const uint32_t x = (uint32_t)__ldg(Sk[k] + (g - pre[k]));
            uint32_t q[3], cd[3];
            int cnt = 0;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const uint32_t v = pi_fwd(t, x);
                q[t] = slot_of(t, v, r, r0, log2r0);
                cd[t] = v >> P.s;
                cnt += (read_byte(k, q[t]) == cd[t]);
            }
            if (cnt == 1)
#pragma unroll
                for (int t = 0; t < 3; ++t) erase(k, q[t], cd[t]);
        }
    }
    if (CS > 1) cg::this_cluster().sync();
    else __syncthreads();
    // encode: b = 1 on the copy whose partner sits in the preceding table (Fig. 5, reading #6);
    // x's bytes are written by x's thread only (plain byte stores)
    for (int g = (int)rank * NT + threadIdx.x; g < ntot; g += CS * NT) {
        int k = 0;
#pragma unroll
        for (int j = 1; j < IPC; ++j) k += (g >= pre[j]);
        const uint32_t x = (uint32_t)__ldg(Sk[k] + (g - pre[k]));
        uint32_t q[3], cd[3];
        bool in[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const uint32_t v = pi_fwd(t, x);
            q[t] = slot_of(t, v, r, r0, log2r0);
            cd[t] = v >> P.s;
            in[t] = read_byte(k, q[t]) == cd[t];
        }
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if (in[t] && !in[(t + 1) % 3]) {
                bool loc;
                const uint32_t a = where(k, q[t], &loc);
                if (loc) sh_st_u8(a, 0x80u | cd[t]);
                else cl_st_u8(a, 0x80u | cd[t]);
            }
    }
    if (CS > 1) cg::this_cluster().sync();
    else __syncthreads();
    // pack: the table words are the arena words (entry e = byte lane e & 3 of word e >> 2)
    if (CS == 1 && stage) {  // each table as one contiguous row of the staging block
        // (k_pack_transpose then writes the arena in 128-byte row segments): one store instruction
        // here moves 512 bytes instead of 32 single words (IPC = 1) or pairs (IPC = 2) n_pad apart
        const uint32_t n16 = slice / 16;
        for (uint32_t i = threadIdx.x; i < (uint32_t)n_it * n16; i += NT) {
            const uint32_t k = i / n16, j = i - k * n16;
            reinterpret_cast<uint4*>(stage + (int64_t)(c0 + k) * (slice / 4))[j] =
                reinterpret_cast<const uint4*>(TB + k * stride_b)[j];
        }
    } else if (IPC == 1) {
        const uint32_t w0 = rank * slice / 4;
        for (uint32_t i = threadIdx.x; i < slice / 16; i += NT) {
            const uint4 v = reinterpret_cast<const uint4*>(TB)[i];
            uint32_t* dst = arena_cls + (int64_t)(w0 + 4 * i) * n_pad + c0;
            dst[0] = v.x;
            dst[(int64_t)n_pad] = v.y;
            dst[2 * (int64_t)n_pad] = v.z;
            dst[3 * (int64_t)n_pad] = v.w;
        }
    } else {  // lane -> (word, item): IPC consecutive columns of a word row per store group
        const uint32_t W = slice / 4;
        for (uint32_t i = threadIdx.x; i < W * IPC; i += NT) {
            const uint32_t w = i / IPC, k = i % IPC;
            if ((int)k < n_it)
                arena_cls[(int64_t)w * n_pad + c0 + k] = *reinterpret_cast<const uint32_t*>(TB + k * stride_b + 4 * w);
        }
    }
    if (CS > 1) cg::this_cluster().sync();  // no CTA may exit while another still reads its slice
}

// Staged pack of the byte tier: stage holds the class's tables item-major ([item][word], W words
// each); the arena block is word-major ([word][n_pad items], the layout K2's TMA boxes read).  A
// 32-item x 32-word tile goes through shared memory: reads of 128 bytes along the words of an item,
// writes of 128 bytes along the items of a word row.
__global__ void __launch_bounds__(256) k_pack_transpose(const uint32_t* __restrict__ stage, int n, uint32_t W,
                                                        uint32_t* __restrict__ arena_cls, int n_pad) {
    __shared__ uint32_t tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, w0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = i0 + ty + 8 * q, w = w0 + tx;
        if (i < n && w < W) tile[ty + 8 * q][tx] = stage[i * W + w];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t w = w0 + ty + 8 * q, i = i0 + tx;
        if (i < n && w < W) arena_cls[w * n_pad + i] = tile[tx][ty + 8 * q];
    }
}

// Encode columns [0, n) of one class block: thread per (word w, column c); writes
// arena_cls[w * n_pad + c] (padding columns are filled by k_fill_padding).
__global__ void __launch_bounds__(256) k1_encode(
    const uint32_t* __restrict__ work, const int64_t* __restrict__ work_off, int64_t first, int n,
    int n_pad, int W, uint32_t r, PiParams P, uint32_t r0, int log2r0,
    uint32_t* __restrict__ arena_cls) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)W * n) return;
    const int w = (int)(idx / n);
    const int c = (int)(idx - (int64_t)w * n);
    const uint32_t* A = work + work_off[first + c];
    const uint4 q4 = *reinterpret_cast<const uint4*>(A + 4 * (int64_t)w);
    const uint32_t xs[4] = {q4.x, q4.y, q4.z, q4.w};
    uint32_t word = 0;
    const uint32_t sb = 3u * r0;
#pragma unroll
    for (int lane = 0; lane < 4; ++lane) {
        const uint32_t x = xs[lane];
        uint32_t byte = kNullByte;
        if (x != kEmpty) {
            const uint32_t q = 4u * (uint32_t)w + lane;
            const int t = (int)((q % sb) >> log2r0);  // table of entry q
            const uint32_t code = pi_eval(P, t, x) >> P.s;  // 7 MSBs of π_t(x)
            const int t1 = (t + 1) % 3;
            const uint32_t q1 = slot_of(t1, pi_eval(P, t1, x), r, r0, log2r0);
            // partner in the following table => this copy precedes it => b = 0;
            // otherwise the partner is in the preceding table => b = 1  (Fig. 5)
            const uint32_t bit = (A[q1] == x) ? 0u : 1u;
            byte = (bit << 7) | code;
        }
        word |= byte << (8 * lane);  // little-endian lanes (reading #17)
    }
    arena_cls[(int64_t)w * n_pad + c] = word;
}

__global__ void k1_check(const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids,
                         int64_t n, int64_t m, int* __restrict__ bad) {
    int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    int lane = threadIdx.x & 31;
    if (item >= n) return;
    int64_t b = offsets[item], e = offsets[item + 1];
    for (int64_t k = b + lane; k < e; k += 32) {
        int32_t t = tids[k];
        if (t < 0 || t >= m || (k > b && tids[k - 1] >= t)) atomicOr(bad, 1);
    }
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }

// ⊥ words in the padding columns [n, n_pad) of a class block (reading #1); every real column is
// written by the build kernels
__global__ void k_fill_padding(uint32_t* __restrict__ arena_cls, int n, int n_pad, int W) {
    const int pad = n_pad - n;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)W * pad) return;
    const int64_t w = idx / pad;
    arena_cls[w * n_pad + n + (idx - w * pad)] = kNullWord;
}

// fail_off[p] = first index of position p in the sorted (pos << 32 | tid) list; f[p] = its count
__global__ void k_fail_offsets(const uint64_t* __restrict__ keys, const int* __restrict__ F_d, int64_t n,
                               int64_t* __restrict__ off, int32_t* __restrict__ f) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p > n) return;
    const int64_t F = *F_d;  // deduplicated count (device: no host round trip)
    auto lb = [&](uint64_t key) {
        int64_t lo = 0, hi = F;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    const int64_t a = lb((uint64_t)p << 32);
    off[p] = a;
    if (p < n) f[p] = (int32_t)(lb((uint64_t)(p + 1) << 32) - a);
}

__global__ void k_fail_split(const uint64_t* __restrict__ keys, const int* __restrict__ F_d, int32_t* __restrict__ tid,
                             int32_t* __restrict__ mark, uint32_t* __restrict__ fbits) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= *F_d) return;
    uint32_t t = (uint32_t)keys[i];
    tid[i] = (int32_t)t;
    mark[t] = 1;
    atomicOr(fbits + (t >> 5), 1u << (t & 31));
}

__global__ void k_fidx(const int32_t* __restrict__ mark, const int32_t* __restrict__ rank, int64_t m,
                       int32_t* __restrict__ fidx) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) fidx[i] = mark[i] ? rank[i] : -1;
}

// Global tier split over CTAs (reading #9b): the giant tables (C4: one item of r = 2^21 holds 1.2e6
// elements) are cut into chunks of kGChunk elements, each chunk a CTA, all inserting concurrently
// into the item's table in L2/HBM with atomic swaps; a chain exceeding MaxLoop records its
// nestless element in F directly.  Copies are conserved by every swap, so once all chunks are done
// an element with exactly one copy left is exactly a recorded failure: k1_gchunk_cleanup deletes
// that copy (F itself is deduplicated and counted per item by post_failures).
constexpr int kGChunk = 2048;
struct GChunk {
    int64_t pos;     // width-sorted position of the item
    int32_t e0, e1;  // element range of the chunk
    int32_t log2r, pad;
};

__global__ void __launch_bounds__(256) k1_gchunk_insert(
    const GChunk* __restrict__ chunks, const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids,
    const int32_t* __restrict__ pos2orig, const int64_t* __restrict__ work_off, int64_t big_begin, PiParams P,
    uint32_t r0, int log2r0, uint32_t max_loop_opt, uint32_t* __restrict__ work, uint64_t* __restrict__ fails,
    unsigned long long* __restrict__ fail_ctr, int64_t fail_cap) {
    const GChunk ch = chunks[blockIdx.x];
    const uint32_t r = 1u << ch.log2r;
    const int32_t* S = tids + offsets[pos2orig[ch.pos]];
    uint32_t* A = work + work_off[ch.pos - big_begin];
    const uint32_t max_loop = max_loop_opt ? max_loop_opt : 16u + 3u * (uint32_t)ch.log2r;
    for (int e = ch.e0 + threadIdx.x; e < ch.e1; e += blockDim.x) {
        const uint32_t x = (uint32_t)__ldg(S + e);
        for (int copy = 0; copy < 2; ++copy) {
            uint32_t tau = x;
            for (uint32_t l = 0; l < max_loop && tau != kEmpty; ++l)
#pragma unroll
                for (int t = 0; t < 3 && tau != kEmpty; ++t)
                    tau = atomicExch(&A[slot_of(t, pi_eval(P, t, tau), r, r0, log2r0)], tau);
            if (tau != kEmpty) {
                const unsigned long long idx = atomicAdd(fail_ctr, 1ull);
                if ((int64_t)idx < fail_cap) fails[idx] = ((uint64_t)ch.pos << 32) | tau;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k1_gchunk_cleanup(
    const GChunk* __restrict__ chunks, const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids,
    const int32_t* __restrict__ pos2orig, const int64_t* __restrict__ work_off, int64_t big_begin, PiParams P,
    uint32_t r0, int log2r0, uint32_t* __restrict__ work) {
    const GChunk ch = chunks[blockIdx.x];
    const uint32_t r = 1u << ch.log2r;
    const int32_t* S = tids + offsets[pos2orig[ch.pos]];
    uint32_t* A = work + work_off[ch.pos - big_begin];
    for (int e = ch.e0 + threadIdx.x; e < ch.e1; e += blockDim.x) {
        const uint32_t x = (uint32_t)__ldg(S + e);
        uint32_t q[3];
        int cnt = 0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            q[t] = slot_of(t, pi_eval(P, t, x), r, r0, log2r0);
            cnt += (A[q[t]] == x);
        }
        if (cnt == 1)
#pragma unroll
            for (int t = 0; t < 3; ++t) atomicCAS(&A[q[t]], x, kEmpty);
    }
}

// Flat over the CSR entries, 4 per thread per step so that the fidx gathers of a thread are
// independent (the pass is latency-bound otherwise).  An entry whose tid failed somewhere
// (fidx >= 0, rare) emits its CSR index and fidx; emits take one cursor atomic per warp.  The item
// of each emitted entry is found afterwards (k_ab_keys), off the scan's critical path.  Writes beyond `cap` are dropped (the caller re-runs
// with the exact count, which the cursor holds either way).
__global__ void __launch_bounds__(256) k_ab_scan(const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids,
                                                 const int32_t* __restrict__ orig2pos, int64_t n, int64_t nnz,
                                                 const int32_t* __restrict__ fidx, const uint32_t* __restrict__ fbits,
                                                 uint64_t* __restrict__ at_k, int32_t* __restrict__ at_f,
                                                 unsigned long long* __restrict__ cursor, int64_t cap) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4 - lane * 4 + lane;
         base - lane < nnz; base += stride) {
        // the warp covers 128 consecutive entries; lane l takes entries base + 32 q (coalesced)
        int32_t f[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t k = base + 32 * q;
            f[q] = -1;
            if (k < nnz) {  // the m-bit set of failed tids is L1-resident; fidx is read for hits only
                const uint32_t t = (uint32_t)__ldg(tids + k);
                if (__ldg(fbits + (t >> 5)) >> (t & 31) & 1u) f[q] = __ldg(fidx + t);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t k = base + 32 * q;
            const bool hit = f[q] >= 0;
            const unsigned mask = __ballot_sync(0xFFFFFFFFu, hit);
            if (!mask) continue;
            unsigned long long at = 0;
            if (lane == __ffs(mask) - 1) at = atomicAdd(cursor, (unsigned long long)__popc(mask));
            at = __shfl_sync(0xFFFFFFFFu, at, __ffs(mask) - 1) + __popc(mask & ((1u << lane) - 1));
            if (hit && (int64_t)at < cap) {
                at_k[at] = (uint64_t)k;
                at_f[at] = f[q];
            }
        }
    }
}

// Sort keys fidx * n + pos of the emitted entries: the item of CSR entry k by binary search in
// offsets (the last item with offsets[item] <= k; empty items are skipped by construction).
__global__ void k_ab_keys(const int64_t* __restrict__ offsets, const int32_t* __restrict__ orig2pos, int64_t n,
                          uint64_t* __restrict__ keys, const int32_t* __restrict__ at_f, int64_t total) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t k = (int64_t)keys[i];
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(offsets + mid) <= k) lo = mid;
        else hi = mid - 1;
    }
    keys[i] = (uint64_t)(uint32_t)at_f[i] * (uint64_t)n + (uint32_t)orig2pos[lo];
}

// A_b from the sorted keys fidx * n + pos: positions, and ab_off[k] = index of failed tid k's first
// key (every failed tid occurs in at least its own item, so each k < nft starts a run), ab_off[nft] =
// total.  One thread per key.
__global__ void k_ab_split(const uint64_t* __restrict__ keys, int64_t total, int64_t n, int64_t nft,
                           int32_t* __restrict__ pos, int64_t* __restrict__ off) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const uint64_t key = keys[i];
    const uint64_t k = key / (uint64_t)n;
    pos[i] = (int32_t)(key - k * (uint64_t)n);
    if (i == 0 || keys[i - 1] / (uint64_t)n != k) off[k] = i;
    if (i == total - 1) off[nft] = total;
}


static inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

static batmap_status cub_tmp(batmap_collection* h, size_t need, cudaStream_t st) {
    if (h->cub_tmp && h->cub_tmp_bytes >= need) return BATMAP_OK;
    dfree(h->cub_tmp, st);
    h->cub_tmp = nullptr;
    size_t b = need + need / 4 + 4096;
    BM_TRY(dalloc(&h->cub_tmp, b, st));
    h->cub_tmp_bytes = b;
    return BATMAP_OK;
}

static int ilog2_u64(uint64_t v) {  // ceil(log2 v), 0 for v <= 1
    return v <= 1 ? 0 : 64 - __builtin_clzll(v - 1);
}

// Failure list F sorted by (pos, tid), per-item offsets and A_b of failed tids.
static batmap_status post_failures(batmap_collection* h, const int64_t* offsets, const int32_t* tids, int64_t nnz,
                                   uint64_t* fails, int64_t F, cudaStream_t st) {
    const int64_t n = h->n, m = h->m;
    BM_TRY(dalloc_t(&h->fail_off_d, n + 1, st));
    BM_TRY(dalloc_t(&h->fidx_of_tid_d, m, st));
    if (F == 0) {
        if (n) BM_CUDA(cudaMemsetAsync(h->f_d, 0, n * sizeof(int32_t), st));
        BM_CUDA(cudaMemsetAsync(h->fail_off_d, 0, (n + 1) * sizeof(int64_t), st));
        k_fill_i32<<<grid_for(m, 256), 256, 0, st>>>(h->fidx_of_tid_d, m, -1);
        h->launches += 1;
        BM_TRY(dalloc_t(&h->fail_tid_d, 1, st));
        BM_TRY(dalloc_t(&h->ab_off_d, 1, st));
        BM_TRY(dalloc_t(&h->ab_pos_d, 1, st));
        BM_CUDA(cudaMemsetAsync(h->ab_off_d, 0, sizeof(int64_t), st));
        h->n_ftid = 0;
        h->n_fail = 0;
        return BATMAP_OK;
    }
    // sort F by (pos, tid) and drop duplicates (the concurrent build may record an element twice)
    uint64_t* sorted = nullptr;
    uint64_t* uniq = nullptr;
    int* n_uniq_d = nullptr;
    int32_t *mark = nullptr, *rank = nullptr;
    uint32_t* fbits = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    int32_t* at_f = nullptr;
    unsigned long long* cursor = nullptr;
    Scratch scratch(st);
    scratch.own(&at_f);
    scratch.own(&sorted);
    scratch.own(&uniq);
    scratch.own(&n_uniq_d);
    scratch.own(&mark);
    scratch.own(&rank);
    scratch.own(&fbits);
    scratch.own(&keys);
    scratch.own(&keys2);
    scratch.own(&cursor);
    BM_TRY(dalloc_t(&sorted, F, st));
    BM_TRY(dalloc_t(&uniq, F, st));
    BM_TRY(dalloc_t(&n_uniq_d, 1, st));
    int end_bit = 32 + std::max(1, ilog2_u64((uint64_t)n + 1));
    {
        size_t tb = 0;
        BM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, fails, sorted, (int)F, 0, end_bit, st));
        BM_TRY(cub_tmp(h, tb, st));
        BM_CUDA(cub::DeviceRadixSort::SortKeys(h->cub_tmp, tb, fails, sorted, (int)F, 0, end_bit, st));
        h->launches += 1;
        tb = 0;
        BM_CUDA(cub::DeviceSelect::Unique(nullptr, tb, sorted, uniq, n_uniq_d, (int)F, st));
        BM_TRY(cub_tmp(h, tb, st));
        BM_CUDA(cub::DeviceSelect::Unique(h->cub_tmp, tb, sorted, uniq, n_uniq_d, (int)F, st));
        h->launches += 1;
    }
    // every size below is bounded by F (before deduplication); the exact counts stay on the device
    // until the one synchronisation before the A_b sort
    std::swap(sorted, uniq);
    // per-item offsets and counts from the deduplicated list
    k_fail_offsets<<<grid_for(n + 1, 256), 256, 0, st>>>(sorted, n_uniq_d, n, h->fail_off_d, h->f_d);
    h->launches += 1;
    BM_TRY(dalloc_t(&h->fail_tid_d, F, st));
    BM_TRY(dalloc_t(&fbits, (m + 31) / 32, st));
    BM_CUDA(cudaMemsetAsync(fbits, 0, (m + 31) / 32 * sizeof(uint32_t), st));
    BM_TRY(dalloc_t(&mark, m + 1, st));
    BM_TRY(dalloc_t(&rank, m + 1, st));
    BM_CUDA(cudaMemsetAsync(mark, 0, (m + 1) * sizeof(int32_t), st));
    k_fail_split<<<grid_for(F, 256), 256, 0, st>>>(sorted, n_uniq_d, h->fail_tid_d, mark, fbits);
    h->launches += 1;
    {
        size_t tb = 0;
        BM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, mark, rank, (int)(m + 1), st));
        BM_TRY(cub_tmp(h, tb, st));
        BM_CUDA(cub::DeviceScan::ExclusiveSum(h->cub_tmp, tb, mark, rank, (int)(m + 1), st));
        h->launches += 1;
    }
    k_fidx<<<grid_for(m, 256), 256, 0, st>>>(mark, rank, m, h->fidx_of_tid_d);
    h->launches += 1;
    // A_b: one pass over the CSR emits (fidx << 32 | pos) for every entry whose tid failed,
    // into a buffer sized by a guess (F failed elements x 4 x the mean item count of a tid); the one
    // synchronisation reads the exact count, and an overflow re-runs the pass at that size
    const unsigned scan_grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(nnz, 1024), 1 << 30));
    int64_t cap = std::max<int64_t>(4096, 4 * F * std::max<int64_t>(1, nnz / std::max<int64_t>(m, 1)) + 1024);
    cap = std::min<int64_t>(cap, std::max<int64_t>(nnz, 1));
    if (const char* e = getenv("BATMAP_AB_CAP")) cap = std::max<int64_t>(1, atoll(e));  // test hook: overflow path
    BM_TRY(dalloc_t(&cursor, 1, st));
    int n_uniq = 0;
    int32_t nft = 0;
    int64_t total = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        BM_TRY(dalloc_t(&keys, cap, st));
        BM_TRY(dalloc_t(&at_f, cap, st));
        BM_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), st));
        k_ab_scan<<<scan_grid, 256, 0, st>>>(offsets, tids, h->orig2pos_d, n, nnz, h->fidx_of_tid_d, fbits, keys,
                                              at_f, cursor, cap);
        h->launches += 1;
        const void* src[3] = {n_uniq_d, rank + m, cursor};
        const size_t bytes[3] = {sizeof(int), sizeof(int32_t), sizeof(int64_t)};
        void* dst[3] = {&n_uniq, &nft, &total};
        BM_TRY(read_scalars(st, 3, src, bytes, dst));
        if (total <= cap) break;
        dfree(keys, st);
        dfree(at_f, st);
        keys = nullptr;
        at_f = nullptr;
        cap = total;
    }
    h->n_fail = n_uniq;
    h->n_ftid = nft;
    k_ab_keys<<<grid_for(total, 256), 256, 0, st>>>(offsets, h->orig2pos_d, n, keys, at_f, total);
    h->launches += 1;
    BM_TRY(dalloc_t(&keys2, total, st));
    {
        const int eb = std::max(1, ilog2_u64((uint64_t)nft * (uint64_t)n));  // keys < nft * n
        size_t tb = 0;
        BM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, (int)total, 0, eb, st));
        BM_TRY(cub_tmp(h, tb, st));
        BM_CUDA(cub::DeviceRadixSort::SortKeys(h->cub_tmp, tb, keys, keys2, (int)total, 0, eb, st));
        h->launches += 1;
    }
    BM_TRY(dalloc_t(&h->ab_off_d, (int64_t)nft + 1, st));
    BM_TRY(dalloc_t(&h->ab_pos_d, total, st));
    k_ab_split<<<grid_for(total, 256), 256, 0, st>>>(keys2, total, n, nft, h->ab_pos_d, h->ab_off_d);
    h->launches += 1;
    return BATMAP_OK;
}

template <int CS, int NT>
static batmap_status launch_cluster(const ClassInfo& c, batmap_collection* h, const int64_t* offsets,
                                    const int32_t* tids, uint64_t* fails, unsigned long long* fail_ctr,
                                    int64_t fail_cap, cudaStream_t st) {
    const size_t smem = (size_t)3 * c.r / CS * sizeof(uint32_t);
    // set on every call: the attribute is per device, and the call is a cheap host-side update
    BM_CUDA(cudaFuncSetAttribute(k1_conc_cluster<CS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kClSliceBytesMax));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)c.n * CS);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // one item per CTA: staged pack as in the byte tier (BATMAP_K1_STAGE=0: direct)
    uint32_t* stage = nullptr;
    const char* se = getenv("BATMAP_K1_STAGE");
    if (CS == 1 && !(se && se[0] == '0') && c.n >= 64 && dalloc_t(&stage, (int64_t)c.n * c.W, st) != BATMAP_OK) {
        stage = nullptr;  // no room for the staging block: pack directly
        cudaGetLastError();
    }
    const batmap_status rc = [&]() -> batmap_status {
        BM_CUDA(cudaLaunchKernelEx(&cfg, k1_conc_cluster<CS, NT>, offsets, tids, (const int32_t*)h->pos2orig_d,
                                   (int64_t)c.first, (uint32_t)c.r, ilog2_u64((uint64_t)c.r), h->pi, (uint32_t)h->r0,
                                   h->log2r0, h->max_loop_opt, h->arena_d + c.word_off, c.n_pad, fails, fail_ctr,
                                   fail_cap, stage));
        h->launches += 1;
        if (stage) {
            const dim3 grid((unsigned)((c.n + 31) / 32), (unsigned)((c.W + 31) / 32));  // x: items, y: words
            k_pack_transpose<<<grid, 256, 0, st>>>(stage, (int)c.n, (uint32_t)c.W, h->arena_d + c.word_off, c.n_pad);
            BM_CUDA(cudaGetLastError());
            h->launches += 1;
        }
        return BATMAP_OK;
    }();
    if (stage) dfree(stage, st);
    return rc;
}

// cluster size: enough CTAs that each holds at most 192 KB of the item's 12r-byte table
static batmap_status launch_cluster_tier(batmap_collection* h, const ClassInfo& c, const int64_t* offsets,
                                         const int32_t* tids, uint64_t* fails, unsigned long long* fail_ctr,
                                         int64_t fail_cap, cudaStream_t st) {
    const int64_t bytes = 12ll * c.r;
    int cs = bytes <= kClSliceBytesMax ? 1 : bytes <= 2ll * kClSliceBytesMax ? 2 : bytes <= 4ll * kClSliceBytesMax ? 4 : 8;
    // a class of few items would leave most SMs idle: spread each item over more CTAs (and threads),
    // which shortens every thread's chain of dependent swaps (C3: 11 items of r = 2^15)
    // (BATMAP_K1_SPREAD=0 keeps the smallest cluster: test hook for every cluster size)
    const char* sp = getenv("BATMAP_K1_SPREAD");
    const bool spread = !(sp && sp[0] == '0');
    while (spread && cs < 8 && (int64_t)c.n * cs * 2 <= h->num_sms) cs *= 2;
    const bool narrow = c.r <= 4096 && cs == 1 && (!spread || c.n >= h->num_sms);
    if (narrow) return launch_cluster<1, 256>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
    if (cs == 1) return launch_cluster<1, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
    if (cs == 2) return launch_cluster<2, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
    if (cs == 4) return launch_cluster<4, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
    return launch_cluster<8, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
}

template <int CS, int IPC, int NT>
static batmap_status launch_byte(const ClassInfo& c, batmap_collection* h, const int64_t* offsets,
                                 const int32_t* tids, uint64_t* fails, unsigned long long* fail_ctr,
                                 int64_t fail_cap, cudaStream_t st) {
    const size_t smem = IPC == 1 ? (size_t)3 * c.r / CS : (size_t)IPC * (3 * c.r + 16);
    BM_CUDA(cudaFuncSetAttribute(k1_byte<CS, IPC, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kByteSliceMax + 256));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((c.n + IPC - 1) / IPC) * CS);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // one or two items per CTA: stage the tables item-major and transpose into the arena (the direct
    // pack's single-word stores n_pad apart cost ~25 % of k1_byte on C5 p = 10 %: build 16.6 -> 12.4
    // ms with staging); BATMAP_K1_STAGE=0: direct
    uint32_t* stage = nullptr;
    const char* se = getenv("BATMAP_K1_STAGE");
    // (IPC = 8 already stores whole 32-byte sectors; BATMAP_K1_STAGE=4 also stages IPC = 4)
    const int stage_max_ipc = se && se[0] == '4' ? 4 : 2;
    if (CS == 1 && IPC <= stage_max_ipc && !(se && se[0] == '0') && c.n >= 64 &&
        dalloc_t(&stage, (int64_t)c.n * c.W, st) != BATMAP_OK) {
        stage = nullptr;  // no room for the staging block: pack directly
        cudaGetLastError();
    }
    const batmap_status rc = [&]() -> batmap_status {
        BM_CUDA(cudaLaunchKernelEx(&cfg, k1_byte<CS, IPC, NT>, offsets, tids, (const int32_t*)h->pos2orig_d,
                                   (int64_t)c.first, (int)c.n, (uint32_t)c.r, ilog2_u64((uint64_t)c.r), h->pi,
                                   (uint32_t)h->r0, h->log2r0, h->max_loop_opt, h->arena_d + c.word_off, c.n_pad,
                                   fails, fail_ctr, fail_cap, stage));
        h->launches += 1;
        if (stage) {
            const dim3 grid((unsigned)((c.n + 31) / 32), (unsigned)((c.W + 31) / 32));  // x: items, y: words
            k_pack_transpose<<<grid, 256, 0, st>>>(stage, (int)c.n, (uint32_t)c.W, h->arena_d + c.word_off, c.n_pad);
            BM_CUDA(cudaGetLastError());
            h->launches += 1;
        }
        return BATMAP_OK;
    }();
    if (stage) dfree(stage, st);
    return rc;
}

// byte tier: the smallest cluster whose CTAs hold <= 192 KB of the item's 3r table bytes, spread over
// more CTAs when the class has too few items to fill the GPU (BATMAP_K1_SPREAD=0 keeps the smallest);
// classes of many small tables put IPC = 2..8 items in one CTA (BATMAP_K1_IPC=1 disables it), so the
// pack stores whole sectors; threads per CTA grow with the table
static batmap_status launch_byte_tier(batmap_collection* h, const ClassInfo& c, const int64_t* offsets,
                                      const int32_t* tids, uint64_t* fails, unsigned long long* fail_ctr,
                                      int64_t fail_cap, cudaStream_t st) {
    const int64_t bytes = 3ll * c.r;
    int cs = 1;
    while (bytes > cs * (int64_t)kByteSliceMax) cs *= 2;
    const char* sp = getenv("BATMAP_K1_SPREAD");
    const bool spread = !(sp && sp[0] == '0');
    while (spread && cs < 8 && (int64_t)c.n * cs * 2 <= h->num_sms) cs *= 2;
    if (cs == 1) {
        const char* ie = getenv("BATMAP_K1_IPC");
        const bool multi = !(ie && ie[0] == '1');
        int ipc = 1;  // items per CTA while the CTAs still fill every SM
        while (multi && ipc < 8 && 2 * ipc * (bytes + 16) <= (int64_t)kByteSliceMax + 256 &&
               (int64_t)c.n >= (int64_t)2 * ipc * h->num_sms)
            ipc *= 2;
        if (ipc == 8) return launch_byte<1, 8, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
        if (ipc == 4) return launch_byte<1, 4, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
        if (ipc == 2) return launch_byte<1, 2, 512>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
        if (bytes <= 24576) return launch_byte<1, 1, 256>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
        if (bytes <= 49152) return launch_byte<1, 1, 512>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
        return launch_byte<1, 1, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
    }
    if (cs == 2) return launch_byte<2, 1, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
    if (cs == 4) return launch_byte<4, 1, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
    return launch_byte<8, 1, 1024>(c, h, offsets, tids, fails, fail_ctr, fail_cap, st);
}

// BATMAP_TRACE=1: host-side timestamps of the build's phases on stderr (diagnostics)
struct HostTrace {
    bool on = false;
    std::chrono::steady_clock::time_point t0, last;
    HostTrace() {
        const char* e = getenv("BATMAP_TRACE");
        on = e && e[0] == '1';
        t0 = last = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[batmap trace] %-28s +%8.3f ms  (at %8.3f ms)\n", what,
                std::chrono::duration<double, std::milli>(now - last).count(),
                std::chrono::duration<double, std::milli>(now - t0).count());
        last = now;
    }
};

batmap_status build_collection(batmap_collection* h, const int64_t* offsets, const int32_t* tids,
                               const batmap_build_opts* o, int part, int n_parts, cudaStream_t st,
                               const int64_t* offsets_host) {
    HostTrace tr;
    const int64_t n = h->n, m = h->m;
    const int64_t l0 = h->launches;
    rec(h, EV_B0, st);
    // ---- parameters (readings #2, #4)
    int s = 0;
    while ((127ll << s) < m) ++s;
    h->s = s;
    h->U = 127ll << s;
    h->pi = make_pi(h->seed, s, o ? o->pi_table : nullptr);

    std::vector<int64_t> off_h(n + 1);
    if (offsets_host) {  // host copy supplied (batmap_mine_host): no read-back, planning overlaps the upload
        std::copy(offsets_host, offsets_host + n + 1, off_h.begin());
    } else if (void* pin = host_staging((size_t)(n + 1) * sizeof(int64_t))) {
        BM_CUDA(cudaMemcpyAsync(pin, offsets, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
        memcpy(off_h.data(), pin, (n + 1) * sizeof(int64_t));
    } else {
        BM_CUDA(cudaMemcpyAsync(off_h.data(), offsets, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        BM_CUDA(cudaStreamSynchronize(st));
    }
    if (off_h[0] != 0) {
        set_error("offsets[0] must be 0");
        return BATMAP_E_INVALID;
    }
    std::vector<uint8_t> lr_item(n);
    const int lmin = std::max(s, ilog2_u64(h->r_min));
    for (int64_t i = 0; i < n; ++i) {
        int64_t sz = off_h[i + 1] - off_h[i];
        if (sz < 0) {
            set_error("offsets must be non-decreasing (item %lld)", (long long)i);
            return BATMAP_E_INVALID;
        }
        if (sz > m) {
            set_error("item %lld has %lld > n_transactions tids", (long long)i, (long long)sz);
            return BATMAP_E_INVALID;
        }
        int l = ilog2_u64((uint64_t)(2 * sz));  // 2^ceil(log2 2|S|)
        lr_item[i] = (uint8_t)std::max(l, lmin);
    }
    tr.mark("offsets read, sizes");
    const int64_t nnz = off_h[n];
    h->nnz = nnz;
    h->size_orig_h.resize(n);
    for (int64_t i = 0; i < n; ++i) h->size_orig_h[i] = (int32_t)(off_h[i + 1] - off_h[i]);
    // ---- sort by width, stable by id (reading #16): counting sort over log2 r
    h->pos2orig_h.resize(n);
    h->orig2pos_h.resize(n);
    {
        int64_t cnt[64] = {0};
        for (int64_t i = 0; i < n; ++i) cnt[lr_item[i]]++;
        int64_t acc = 0;
        for (int l = 0; l < 64; ++l) {
            int64_t c = cnt[l];
            cnt[l] = acc;
            acc += c;
        }
        for (int64_t i = 0; i < n; ++i) {
            int64_t p = cnt[lr_item[i]]++;
            h->pos2orig_h[p] = (int32_t)i;
            h->orig2pos_h[i] = (int32_t)p;
        }
    }
    std::vector<uint8_t> lr_pos(n);
    for (int64_t p = 0; p < n; ++p) lr_pos[p] = lr_item[h->pos2orig_h[p]];
    h->arena_bytes_raw = 0;
    h->classes.clear();
    std::vector<int> class_maxS;
    std::vector<int64_t> class_sumS;
    int64_t word_off = 0;
    for (int64_t p = 0; p < n;) {
        int64_t q = p;
        int maxS = 0;
        int64_t sumS = 0;
        while (q < n && lr_pos[q] == lr_pos[p]) {
            const int32_t o2 = h->pos2orig_h[q];
            maxS = std::max<int>(maxS, (int)(off_h[o2 + 1] - off_h[o2]));
            sumS += off_h[o2 + 1] - off_h[o2];
            ++q;
        }
        ClassInfo c{};
        c.first = p;
        c.n = (int32_t)(q - p);
        c.n_pad = (int32_t)((c.n + kPadItems - 1) / kPadItems * kPadItems);
        c.r = 1 << lr_pos[p];
        c.W = 3 * c.r / 4;
        c.word_off = word_off;
        word_off += (int64_t)c.W * c.n_pad;
        h->arena_bytes_raw += 3ll * c.r * c.n;
        h->classes.push_back(c);
        class_maxS.push_back(maxS);
        class_sumS.push_back(sumS);
        p = q;
    }
    h->arena_words = word_off;
    h->r0 = n ? (1ll << lr_pos[0]) : (1ll << lmin);  // r0 = min r_i (reading #5)
    h->log2r0 = ilog2_u64((uint64_t)h->r0);
    if (h->arena_words > (1ll << 40)) {
        set_error("arena too large");
        return BATMAP_E_OVERFLOW;
    }
    // the intersection's host plan (C4: 3e5 work items, milliseconds of host time) is made on a worker
    // thread while this build's kernels run; prepare_full_k2 uploads it once K1 is launched.  Small
    // plans are made inline (a thread costs more than they do).
    struct PlanTask {
        std::future<K2Prepared*> f;
        cudaStream_t st;
        ~PlanTask() {
            if (f.valid()) destroy_k2(f.get(), st);  // early error return: drop the unused plan
        }
    } plan_task{{}, st};
    if (n >= 16384 && full_k2_plannable(h))
        plan_task.f = std::async(std::launch::async, new_k2_host_plan, h->classes, h->num_sms, part, n_parts);
    // items of classes with r > glob_min_r (the last positions) use a working table in global memory
    const bool serial = o && (o->flags & BATMAP_BUILD_SERIAL);
    // concurrent tiers: the byte-table kernel (k1_byte, r <= 2^19) unless disabled or a test π
    // table is supplied (the byte tier inverts the hash form of π); else the uint32 cluster kernel
    // (BATMAP_K1_BYTE=0: never; =all: every class up to 2^19, clusters included -- test hooks).  By
    // default (measured, profiles/r2_k1_tiers.jsonl): tables of <= 192 KB as bytes (r <= 2^16) that
    // would need a cluster as uint32 (r >= 2^15), and classes of many nearly empty tables (C4: ~13
    // elements in r = 8192), whose cost is the pack and which the byte tier packs 8 items at a time;
    // denser narrow tables stay in the uint32 kernel (fewer instructions per swap); r > 2^16 goes to
    // the global tier, which spreads a few giant items over many CTAs.
    const char* bt_env = getenv("BATMAP_K1_BYTE");
    const int byte_mode = serial || h->pi.table != nullptr || (bt_env && bt_env[0] == '0') ? 0
                          : (bt_env && bt_env[0] == 'a') ? 2 : 1;
    auto use_byte = [&](size_t a) {
        const ClassInfo& c = h->classes[a];
        if (byte_mode != 1) return byte_mode == 2;
        if (c.r > 16384) return true;
        return class_sumS[a] * 16 < (int64_t)c.n * c.r && (int64_t)c.n >= 4ll * h->num_sms;
    };
    const int64_t glob_min_r =
        serial ? kSmallMaxR : byte_mode == 2 ? (int64_t)kByteMaxR : byte_mode == 1 ? 65536 : (int64_t)kClusterMaxR;
    int64_t big_begin = n;
    for (const ClassInfo& c : h->classes)
        if (c.r > glob_min_r) {
            big_begin = c.first;
            break;
        }
    const int64_t n_big = n - big_begin;
    std::vector<int64_t> work_off(n_big + 1, 0);
    for (int64_t p = 0; p < n_big; ++p) work_off[p + 1] = work_off[p] + 3ll * (1ll << lr_pos[big_begin + p]);
    const int64_t work_entries = work_off[n_big];

    // sharded build: class a is cut into n_parts column chunks; part p builds chunk
    // (p + rot[a]) mod n_parts.  The rotations deal the chunks by estimated insertion cost, greedily,
    // most expensive class first, so that parts receiving a giant item get fewer of the cheap ones
    // (every rank computes the same rotations from the same tidlist sizes).
    h->shard_rot.assign(h->classes.size(), 0);
    if (n_parts > 1) {
        std::vector<std::vector<double>> chunk(h->classes.size(), std::vector<double>(n_parts, 0.0));
        std::vector<std::pair<double, size_t>> order;
        for (size_t a = 0; a < h->classes.size(); ++a) {
            const ClassInfo& c = h->classes[a];
            for (int j = 0; j < n_parts; ++j) {
                const int64_t q0 = (int64_t)c.n * j / n_parts, q1 = (int64_t)c.n * (j + 1) / n_parts;
                for (int64_t q = q0; q < q1; ++q) {
                    const int32_t o2 = h->pos2orig_h[c.first + q];
                    // ~ 60 bytes of arena traffic per insertion (profiles/r2_k1_tiers.jsonl)
                    chunk[a][j] += 120.0 * (double)(off_h[o2 + 1] - off_h[o2]) + 3.0 * c.r;
                }
            }
            order.push_back({*std::max_element(chunk[a].begin(), chunk[a].end()), a});
        }
        std::stable_sort(order.begin(), order.end(), [](const std::pair<double, size_t>& x,
                                                        const std::pair<double, size_t>& y) { return x.first > y.first; });
        std::vector<double> load(n_parts, 0.0);
        for (const auto& oa : order) {
            const size_t a = oa.second;
            int best = 0;
            double best_max = 0.0;
            for (int o = 0; o < n_parts; ++o) {
                double mx = 0.0;
                for (int p = 0; p < n_parts; ++p) mx = std::max(mx, load[p] + chunk[a][(p + o) % n_parts]);
                if (o == 0 || mx < best_max) {
                    best = o;
                    best_max = mx;
                }
            }
            h->shard_rot[a] = best;
            for (int p = 0; p < n_parts; ++p) load[p] += chunk[a][(p + best) % n_parts];
        }
    }
    // this part's share of every class (the whole class when n_parts == 1)
    auto view = [&](const ClassInfo& c) {
        ClassInfo v = c;
        int64_t c0, c1;
        shard_cols(h, (size_t)(&c - h->classes.data()), part, n_parts, &c0, &c1);
        v.first = c.first + c0;
        v.n = (int32_t)(c1 - c0);
        v.word_off = c.word_off + c0;
        return v;
    };
    // ---- chunks of the global tier's items (this part's share of each class)
    std::vector<GChunk> gchunks;
    if (!serial)
        for (const ClassInfo& cl : h->classes) {
            const ClassInfo c = view(cl);
            if (c.r <= glob_min_r) continue;
            for (int64_t p = c.first; p < c.first + c.n; ++p) {
                const int32_t o2 = h->pos2orig_h[p];
                const int32_t len = (int32_t)(off_h[o2 + 1] - off_h[o2]);
                for (int32_t e0 = 0; e0 < std::max(len, 1); e0 += kGChunk)
                    gchunks.push_back({p, e0, std::min(len, e0 + kGChunk), ilog2_u64((uint64_t)c.r), 0});
            }
        }
    tr.mark("sort, classes, chunks");
    // ---- device state
    BM_TRY(dalloc_t(&h->pos2orig_d, n, st));
    BM_TRY(dalloc_t(&h->orig2pos_d, n, st));
    BM_TRY(dalloc_t(&h->f_d, n, st));
    BM_TRY(dalloc_t(&h->arena_d, h->arena_words, st));
    int64_t* work_off_d = nullptr;
    uint8_t* lr_d = nullptr;
    uint32_t* work = nullptr;
    GChunk* gchunks_d = nullptr;
    uint64_t* fails = nullptr;
    unsigned long long* fail_ctr = nullptr;
    int* bad = nullptr;
    Scratch scratch(st);
    scratch.own(&work_off_d);
    scratch.own(&lr_d);
    scratch.own(&work);
    scratch.own(&gchunks_d);
    scratch.own(&fails);
    scratch.own(&fail_ctr);
    scratch.own(&bad);
    BM_TRY(dalloc_t(&work_off_d, n_big + 1, st));
    BM_TRY(dalloc_t(&lr_d, n, st));
    BM_TRY(dalloc_t(&work, work_entries, st));
    BM_TRY(dalloc_t(&gchunks_d, (int64_t)gchunks.size(), st));
    {  // host tables -> device, staged through pinned memory (asynchronous copies)
        struct Up {
            void* dst;
            const void* src;
            size_t bytes;
        };
        const Up ups[5] = {{gchunks_d, gchunks.data(), gchunks.size() * sizeof(GChunk)},
                           {h->pos2orig_d, h->pos2orig_h.data(), (size_t)n * 4},
                           {h->orig2pos_d, h->orig2pos_h.data(), (size_t)n * 4},
                           {work_off_d, work_off.data(), n ? (size_t)(n_big + 1) * 8 : 0},
                           {lr_d, lr_pos.data(), (size_t)n}};
        size_t total = 0;
        for (const Up& u : ups) total += (u.bytes + 15) / 16 * 16;
        char* pin = static_cast<char*>(host_staging(total));
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
    }
    tr.mark("allocs + uploads");
    if (o && (o->flags & BATMAP_CHECK_INPUT) && n) {
        BM_TRY(dalloc_t(&bad, 1, st));
        BM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
        k1_check<<<grid_for(n * 32, 256), 256, 0, st>>>(offsets, tids, n, m, bad);
        h->launches += 1;
        int bad_h = 0;
        BM_TRY(read_scalar(st, bad, &bad_h));
        if (bad_h) {
            set_error("invalid tidlists: every tidlist must be strictly increasing in [0, n_transactions)");
            return BATMAP_E_INVALID;
        }
    }
    // failure buffer: generous first guess, exact retry if exceeded (the build is deterministic)
    int64_t fail_cap = std::max<int64_t>(1 << 16, nnz / 16);
    BM_TRY(dalloc_t(&fail_ctr, 1, st));
    int64_t F = 0;
    // per device (no process-wide flag: a process may drive several GPUs)
    BM_CUDA(cudaFuncSetAttribute(k1_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    BM_CUDA(cudaFuncSetAttribute(k1_conc_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int attempt = 0; attempt < 4; ++attempt) {
        BM_TRY(dalloc_t(&fails, fail_cap, st));
        for (const ClassInfo& c : h->classes) {  // ⊥ padding
            const int64_t cnt = (int64_t)c.W * (c.n_pad - c.n);
            if (cnt == 0) continue;
            k_fill_padding<<<grid_for(cnt, 256), 256, 0, st>>>(h->arena_d + c.word_off, c.n, c.n_pad, c.W);
            h->launches += 1;
        }
        if (work_entries) BM_CUDA(cudaMemsetAsync(work, 0xFF, work_entries * sizeof(uint32_t), st));
        BM_CUDA(cudaMemsetAsync(fail_ctr, 0, sizeof(unsigned long long), st));
        rec(h, EV_I0, st);
        if (serial) {
            for (size_t a = 0; a < h->classes.size(); ++a) {  // launched first: long serial chains overlap
                const ClassInfo c = view(h->classes[a]);
                if (c.r <= kSmallMaxR || c.n == 0) continue;
                k1_insert<<<grid_for(c.n, 32), 32, 0, st>>>(offsets, tids, h->pos2orig_d,
                                                            work_off_d + (c.first - big_begin), lr_d, c.first, c.n,
                                                            h->pi, (uint32_t)h->r0, h->log2r0, h->max_loop_opt, work,
                                                            h->f_d, fails, fail_ctr, fail_cap);
                h->launches += 1;
            }
            for (size_t a = 0; a < h->classes.size(); ++a) {
                const ClassInfo c = view(h->classes[a]);
                if (c.r > kSmallMaxR || c.n == 0) continue;
                const int maxS = std::max(class_maxS[a], 1);
                const size_t smem = (size_t)6 * c.r + (size_t)9 * maxS + 16;
                k1_small<<<c.n, 32, smem, st>>>(offsets, tids, h->pos2orig_d, c.first, c.W, (uint32_t)c.r,
                                                ilog2_u64((uint64_t)c.r), maxS, h->pi, (uint32_t)h->r0, h->log2r0,
                                                h->max_loop_opt, h->arena_d + c.word_off, c.n_pad, h->f_d, fails,
                                                fail_ctr, fail_cap);
                h->launches += 1;
            }
        } else {
            if (!gchunks.empty()) {  // big classes first (longest items), split over CTAs
                k1_gchunk_insert<<<(unsigned)gchunks.size(), 256, 0, st>>>(
                    gchunks_d, offsets, tids, h->pos2orig_d, work_off_d, big_begin, h->pi, (uint32_t)h->r0,
                    h->log2r0, h->max_loop_opt, work, fails, fail_ctr, fail_cap);
                h->launches += 1;
            }
            // r <= cl_min_r: the slot-caching CTA kernel (faster for narrow tables, measured on C2);
            // wider tables: the cluster kernel.  BATMAP_K1_SMALL=legacy|cluster moves the boundary.
            const int64_t cl_min_r = [] {  // read per build (tests switch it)
                const char* v = getenv("BATMAP_K1_SMALL");
                if (v && v[0] == 'l') return (int64_t)kSmallMaxR;
                if (v && v[0] == 'c') return (int64_t)0;
                return (int64_t)2048;
            }();
            // classes of few items (a grid smaller than the GPU) run on a side stream beside the
            // many-item classes, so that they fill the SMs the others' partial waves leave idle
            // (C3 build 0.56 -> 0.50 ms); BATMAP_K1_SIDE=0 keeps one stream
            constexpr int kMaxDev = 64;
            static thread_local cudaStream_t side_of[kMaxDev] = {};
            static thread_local cudaEvent_t fork_of[kMaxDev] = {}, join_of[kMaxDev] = {};
            const char* se = getenv("BATMAP_K1_SIDE");
            bool any_few = false, any_many = false;
            for (const ClassInfo& cl : h->classes) {
                const ClassInfo c = view(cl);
                if (c.n == 0 || c.r > glob_min_r) continue;
                (c.n < h->num_sms ? any_few : any_many) = true;
            }
            const bool use_side = !(se && se[0] == '0') && any_few && any_many && h->device < kMaxDev;
            cudaStream_t side = nullptr;
            // joins the side stream back into st on every exit from this scope, so that nothing
            // freed or read on st afterwards can race the side stream's kernels
            struct Join {
                cudaStream_t side = nullptr, st = nullptr;
                cudaEvent_t ev = nullptr;
                ~Join() {
                    if (side && cudaEventRecord(ev, side) == cudaSuccess) cudaStreamWaitEvent(st, ev, 0);
                }
            } join;
            if (use_side) {
                const int d = h->device;
                if (!side_of[d]) {
                    BM_CUDA(cudaStreamCreateWithFlags(&side_of[d], cudaStreamNonBlocking));
                    BM_CUDA(cudaEventCreateWithFlags(&fork_of[d], cudaEventDisableTiming));
                    BM_CUDA(cudaEventCreateWithFlags(&join_of[d], cudaEventDisableTiming));
                }
                side = side_of[d];
                BM_CUDA(cudaEventRecord(fork_of[d], st));
                BM_CUDA(cudaStreamWaitEvent(side, fork_of[d], 0));
                join.side = side;
                join.st = st;
                join.ev = join_of[d];
            }
            auto sfor = [&](const ClassInfo& c) { return use_side && c.n < h->num_sms ? side : st; };
            for (size_t a = h->classes.size(); a-- > 0;) {  // cluster tier, widest first
                const ClassInfo c = view(h->classes[a]);
                if (c.r <= cl_min_r || c.r > glob_min_r || c.n == 0) continue;
                if (use_byte(a)) BM_TRY(launch_byte_tier(h, c, offsets, tids, fails, fail_ctr, fail_cap, sfor(c)));
                else BM_TRY(launch_cluster_tier(h, c, offsets, tids, fails, fail_ctr, fail_cap, sfor(c)));
            }
            for (size_t a = 0; a < h->classes.size(); ++a) {
                const ClassInfo c = view(h->classes[a]);
                if (c.r > cl_min_r || c.n == 0) continue;
                const int maxS = std::max(class_maxS[a], 1);
                const size_t smem = (size_t)12 * c.r + (size_t)9 * maxS + 16;
                k1_conc_small<<<c.n, kConcThreads, smem, sfor(c)>>>(
                    offsets, tids, h->pos2orig_d, c.first, c.W, (uint32_t)c.r, ilog2_u64((uint64_t)c.r), maxS, h->pi,
                    (uint32_t)h->r0, h->log2r0, h->max_loop_opt, h->arena_d + c.word_off, c.n_pad, h->f_d, fails,
                    fail_ctr, fail_cap);
                h->launches += 1;
            }
        }
        if (!serial && !gchunks.empty()) {
            k1_gchunk_cleanup<<<(unsigned)gchunks.size(), 256, 0, st>>>(gchunks_d, offsets, tids, h->pos2orig_d,
                                                                        work_off_d, big_begin, h->pi,
                                                                        (uint32_t)h->r0, h->log2r0, work);
            h->launches += 1;
        }
        rec(h, EV_I1, st);
        BM_CUDA(cudaGetLastError());
        tr.mark("K1 launched");
        // plan the intersection of the full selection on the host while the build kernels run
        if (attempt == 0) {
            K2Prepared* hp = plan_task.f.valid() ? plan_task.f.get() : nullptr;
            tr.mark("host plan joined");
            BM_TRY(prepare_full_k2(h, part, n_parts, st, hp));
            tr.mark("plan uploaded");
        }
        unsigned long long Fh = 0;
        BM_TRY(read_scalar(st, fail_ctr, &Fh));
        tr.mark("K1 done (sync)");
        F = (int64_t)Fh;
        if (F <= fail_cap) break;
        dfree(fails, st);
        fails = nullptr;
        fail_cap = 2 * F + 1024;  // the concurrent build is not deterministic: leave headroom
    }
    if (F > fail_cap || fails == nullptr) {  // every attempt overflowed: never read an undersized list
        set_error("build: %lld failed insertions exceed the failure buffer after 4 attempts", (long long)F);
        return BATMAP_E_CAPACITY;
    }
    h->n_fail = F;
    rec(h, EV_E0, st);
    for (const ClassInfo& cl : h->classes) {
        const ClassInfo c = view(cl);
        if (c.r <= glob_min_r || c.n == 0) continue;
        int64_t cnt = (int64_t)c.W * c.n;
        k1_encode<<<grid_for(cnt, 256), 256, 0, st>>>(work, work_off_d, c.first - big_begin, c.n, c.n_pad, c.W,
                                                      (uint32_t)c.r, h->pi, (uint32_t)h->r0, h->log2r0,
                                                      h->arena_d + c.word_off);
        h->launches += 1;
    }
    rec(h, EV_E1, st);
    BM_CUDA(cudaGetLastError());
    if (n_parts == 1) {
        BM_TRY(post_failures(h, offsets, tids, nnz, fails, F, st));
    } else {  // sharded: keep this part's failure records for the exchange (batmap_shard_import)
        BM_TRY(dalloc_t(&h->shard_fails_d, std::max<int64_t>(F, 1), st));
        if (F) BM_CUDA(cudaMemcpyAsync(h->shard_fails_d, fails, F * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
        h->shard_n_fail = F;
        h->shard_part = part;
        h->shard_n_parts = n_parts;
        h->shard_pending = true;
    }
    BM_CUDA(cudaGetLastError());
    rec(h, EV_B1, st);  // the scratch buffers are freed on return
    tr.mark("encode + post queued");
    h->build_timed = true;
    h->stats.launches_build = h->launches - l0;
    return BATMAP_OK;
}

// Words of part p's share of the arena (all classes, in class order, each [W][c1 - c0]).
void shard_cols(const batmap_collection* h, size_t a, int p, int n_parts, int64_t* c0, int64_t* c1) {
    const int64_t n = h->classes[a].n;
    const int j = n_parts > 1 && a < h->shard_rot.size() ? (p + h->shard_rot[a]) % n_parts : p;
    *c0 = n * j / n_parts;
    *c1 = n * (j + 1) / n_parts;
}

int64_t shard_words(const batmap_collection* h, int p, int n_parts) {
    int64_t words = 0;
    for (size_t a = 0; a < h->classes.size(); ++a) {
        int64_t c0, c1;
        shard_cols(h, a, p, n_parts, &c0, &c1);
        words += (c1 - c0) * h->classes[a].W;
    }
    return words;
}

// Copy part p's columns between the arena and a packed [class][W][cols] buffer (2-D DMA copies).
batmap_status shard_copy(batmap_collection* h, int p, int n_parts, uint32_t* packed, bool to_arena,
                         cudaStream_t st) {
    int64_t off = 0;
    for (size_t ci = 0; ci < h->classes.size(); ++ci) {
        const ClassInfo& c = h->classes[ci];
        int64_t c0, c1;
        shard_cols(h, ci, p, n_parts, &c0, &c1);
        if (c1 == c0) continue;
        uint32_t* a = h->arena_d + c.word_off + c0;
        uint32_t* b = packed + off;
        const size_t wb = (size_t)(c1 - c0) * 4, pitch_a = (size_t)c.n_pad * 4;
        if (to_arena)
            BM_CUDA(cudaMemcpy2DAsync(a, pitch_a, b, wb, wb, (size_t)c.W, cudaMemcpyDeviceToDevice, st));
        else
            BM_CUDA(cudaMemcpy2DAsync(b, wb, a, pitch_a, wb, (size_t)c.W, cudaMemcpyDeviceToDevice, st));
        off += (c1 - c0) * c.W;
    }
    return BATMAP_OK;
}

// Complete a sharded build: the other parts' columns into the arena, then F, f, Fail(i) and A_b
// from every part's failure records exactly as after a whole build.
batmap_status shard_import(batmap_collection* h, const int64_t* offsets, const int32_t* tids,
                           const uint32_t* words_all, int64_t stride_words, const uint64_t* fails_all,
                           const int64_t* n_fails, int64_t stride_fails, cudaStream_t st) {
    const int N = h->shard_n_parts;
    for (int p = 0; p < N; ++p) {
        if (p == h->shard_part) continue;
        BM_TRY(shard_copy(h, p, N, const_cast<uint32_t*>(words_all) + (int64_t)p * stride_words, true, st));
    }
    int64_t F = 0;
    for (int p = 0; p < N; ++p) F += n_fails[p];
    uint64_t* fails = nullptr;
    Scratch scratch(st);
    scratch.own(&fails);
    BM_TRY(dalloc_t(&fails, std::max<int64_t>(F, 1), st));
    int64_t at = 0;
    for (int p = 0; p < N; ++p) {
        if (n_fails[p] == 0) continue;
        BM_CUDA(cudaMemcpyAsync(fails + at, fails_all + (int64_t)p * stride_fails, n_fails[p] * sizeof(uint64_t),
                                cudaMemcpyDeviceToDevice, st));
        at += n_fails[p];
    }
    BM_TRY(post_failures(h, offsets, tids, h->nnz, fails, F, st));
    dfree(h->shard_fails_d, st);
    h->shard_fails_d = nullptr;
    h->shard_pending = false;
    BM_CUDA(cudaGetLastError());
    return BATMAP_OK;
}

}  // namespace bm
