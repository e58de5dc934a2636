// merge.cu -- NEXT-2 comparison path: the same thresholded pair supports by
// sorted-list merging, the classical intersection the paper measures BatMaps against
// (a two-finger merge of two sorted lists of lengths a and b takes
// a + b steps).  Not the BatMap method.
//
// B200 shape: a CTA takes one row item i and 256 column items j > i; S_i is staged once in
// shared memory, and each warp intersects S_i with its 32 column lists one at a time, S_j staged
// by a coalesced copy.  The 32 lanes split the merge of the pair along its merge path (the
// diagonal d = lane * (a+b)/32 is located by a binary search, ties taking S_i first), so every
// lane runs (a+b)/32 two-finger steps; a common element is counted by the lane that consumes its
// S_j copy, whose predecessor in the merge is the S_i copy.  A step is one shared-memory load and
// ~10 integer instructions, branch-free -- the kernel is issue-bound.
#include <algorithm>

#include "common.cuh"

namespace bm {

constexpr int kMergeThreads = 256;
constexpr int kMergeWarps = kMergeThreads / 32;
constexpr int32_t kInf = 0x7FFFFFFF;  // above every tid (tids < 2^31 - 1)

__device__ __forceinline__ int32_t lds32(uint32_t addr) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// Two-finger steps d0 .. d1 of the merge path from (p, q), branch-free; lists
// end in a kInf sentinel.  Counts the S_j elements whose merge predecessor is an equal S_i element.
// kA / kB: the list is in shared memory (else global, read through L1/L2).
template <bool kA, bool kB>
__device__ __forceinline__ int32_t ld_list(bool takeA, uint32_t sa, uint32_t sb, const int32_t* ga,
                                           const int32_t* gb) {
    if (kA && kB) return lds32(takeA ? sa : sb);
    if (takeA) return kA ? lds32(sa) : __ldg(ga);
    return kB ? lds32(sb) : __ldg(gb);
}

template <bool kA, bool kB>
__device__ __forceinline__ uint32_t merge_steps_run(const int32_t* A, const int32_t* B, int p, int q, int steps) {
    uint32_t cnt = 0;
    int32_t lastA = p > 0 ? A[p - 1] : -1;
    int32_t x = A[p], y = B[q];
    uint32_t sa = kA ? (uint32_t)__cvta_generic_to_shared(A + p) : 0u;
    uint32_t sb = kB ? (uint32_t)__cvta_generic_to_shared(B + q) : 0u;
    const int32_t* ga = A + p;
    const int32_t* gb = B + q;
    for (int d = 0; d < steps; ++d) {
        const bool takeA = x <= y;
        cnt += (!takeA && y == lastA);
        lastA = takeA ? x : lastA;
        if (kA) sa += takeA ? 4u : 0u;
        else ga += takeA;
        if (kB) sb += takeA ? 0u : 4u;
        else gb += !takeA;
        const int32_t nv = ld_list<kA, kB>(takeA, sa, sb, ga, gb);
        x = takeA ? nv : x;
        y = takeA ? y : nv;
    }
    return cnt;
}

// kA: S_i staged in shared memory (up to cap_a - 1 elements + a kInf sentinel); kB: every S_j
// staged per warp (up to cap_b - 1 + sentinel).  A list not staged is read through L1/L2 from the
// sentinel-padded copy of the CSR `tids_pad` (list k at offsets[k] + k).
template <bool kA, bool kB>
__global__ void __launch_bounds__(kMergeThreads) k_merge(const int64_t* __restrict__ offsets,
                                                         const int32_t* __restrict__ tids,
                                                         const int32_t* __restrict__ tids_pad, int cap_a,
                                                         const int32_t* __restrict__ sel, int64_t n_sel,
                                                         const int2* __restrict__ tasks, int cap_b, uint32_t thr,
                                                         uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                         unsigned long long* __restrict__ ctr, int64_t cap) {
    extern __shared__ __align__(16) int32_t msm[];
    const int2 tk = tasks[blockIdx.x];
    const int64_t s = tk.x;
    const int ia = sel ? sel[s] : (int)s;
    const int64_t a0 = offsets[ia];
    const int a = (int)(offsets[ia + 1] - a0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t* Si = msm;                                        // S_i (+ sentinel)
    int32_t* Bw = msm + (kA ? cap_a : 0) + warp * cap_b;      // this warp's S_j (+ sentinel)
    if (kA) {
        for (int k = threadIdx.x; k < a; k += kMergeThreads) Si[k] = __ldg(tids + a0 + k);
        if (threadIdx.x == 0) Si[a] = kInf;
    }
    __syncthreads();
    const int32_t* A = kA ? Si : tids_pad + a0 + ia;
    for (int c = 0; c < 32; ++c) {
        const int64_t t = (int64_t)tk.y * kMergeThreads + warp * 32 + c;
        if (t <= s || t >= n_sel) continue;  // warp-uniform
        const int jb = sel ? sel[t] : (int)t;
        const int64_t b0 = offsets[jb];
        const int b = (int)(offsets[jb + 1] - b0);
        const int32_t* B = tids_pad + b0 + jb;
        if (kB) {
            __syncwarp();
            for (int k = lane; k < b; k += 32) Bw[k] = __ldg(tids + b0 + k);
            if (lane == 0) Bw[b] = kInf;
            __syncwarp();
            B = Bw;
        }
        // this lane's part of the merge path: diagonals [d0, d1)
        const int total = a + b;
        const int L = (total + 31) >> 5;
        const int d0 = min(lane * L, total), d1 = min(d0 + L, total);
        int lo = max(0, d0 - b), hi = min(d0, a);
        while (lo < hi) {  // p = #S_i elements among the first d0 merged (ties: S_i first)
            const int mid = (lo + hi) >> 1;
            if (A[mid] <= B[d0 - 1 - mid]) lo = mid + 1;
            else hi = mid;
        }
        uint32_t cnt = merge_steps_run<kA, kB>(A, B, lo, d0 - lo, d1 - d0);
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0 && cnt >= thr) {
            uint32_t u = (uint32_t)ia, v = (uint32_t)jb;
            if (u > v) {
                const uint32_t w = u;
                u = v;
                v = w;
            }
            const unsigned long long at = atomicAdd(ctr, 1ull);
            if ((int64_t)at < cap) {
                keys[at] = ((uint64_t)u << 32) | v;
                vals[at] = cnt;
            }
        }
    }
}

// Sentinel-padded copy of the CSR for the global-memory variant: list k at pad_off[k] + k.
__global__ void k_pad_lists(const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids, int64_t n,
                            int32_t* __restrict__ out) {
    const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (item >= n) return;
    const int64_t b = offsets[item], e = offsets[item + 1];
    for (int64_t k = b + lane; k < e; k += 32) out[k + item] = tids[k];
    if (lane == 0) out[e + item] = kInf;
}

batmap_status merge_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items, const int32_t* items,
                                  int64_t n_sel, uint32_t threshold, batmap_triple* out, int64_t capacity,
                                  int64_t* n_out, double* kernel_ms, int64_t* merge_steps, cudaStream_t st) {
    const int64_t ns = items ? n_sel : n_items;
    *n_out = 0;
    if (kernel_ms) *kernel_ms = 0;
    if (merge_steps) *merge_steps = 0;
    if (ns < 2) return BATMAP_OK;
    // list lengths of the selection (host): staging size, task list, algorithmic step count
    std::vector<int64_t> off(n_items + 1);
    BM_CUDA(cudaMemcpyAsync(off.data(), offsets, (n_items + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> sel_h;
    if (items) {
        sel_h.resize(ns);
        BM_CUDA(cudaMemcpyAsync(sel_h.data(), items, ns * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    }
    BM_CUDA(cudaStreamSynchronize(st));
    int64_t max_len = 0, sum_len = 0;
    for (int64_t k = 0; k < ns; ++k) {
        const int64_t id = items ? sel_h[k] : k;
        const int64_t len = off[id + 1] - off[id];
        max_len = std::max(max_len, len);
        sum_len += len;
    }
    if (merge_steps) *merge_steps = (ns - 1) * sum_len;  // sum over pairs of (a + b)
    std::vector<int2> task;
    const int64_t nb = (ns + kMergeThreads - 1) / kMergeThreads;
    for (int64_t s = 0; s + 1 < ns; ++s)
        for (int64_t cb = (s + 1) / kMergeThreads; cb < nb; ++cb) task.push_back(make_int2((int)s, (int)cb));
    const size_t smem_max = 200 * 1024;
    const int cap = (int)(max_len + 1);  // + the kInf sentinel
    // both lists staged in shared memory, or neither: a step that loads from shared memory in some
    // lanes and from global memory in others issues both loads (measured 2x slower on C3)
    const bool stage_b = (size_t)(kMergeWarps + 1) * cap * 4 <= smem_max;
    const size_t smem = stage_b ? (size_t)(kMergeWarps + 1) * cap * 4 : 0;
    BM_CUDA(cudaFuncSetAttribute(k_merge<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
    int2* task_d = nullptr;
    int32_t* tids_pad = nullptr;
    uint64_t* keys = nullptr;
    uint32_t* vals = nullptr;
    unsigned long long* ctr = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int64_t kcap = std::max<int64_t>(1 << 20, 16 * ns);
    batmap_status rc = BATMAP_OK;
    auto cleanup = [&]() {
        dfree(task_d, st);
        dfree(tids_pad, st);
        dfree(keys, st);
        dfree(vals, st);
        dfree(ctr, st);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    };
    if ((rc = dalloc_t(&task_d, (int64_t)task.size(), st)) != BATMAP_OK || (rc = dalloc_t(&ctr, 1, st)) != BATMAP_OK) {
        cleanup();
        return rc;
    }
    if (!stage_b) {  // lists read from global memory: sentinel-padded copy
        if ((rc = dalloc_t(&tids_pad, off[n_items] + n_items, st)) != BATMAP_OK) {
            cleanup();
            return rc;
        }
        k_pad_lists<<<(unsigned)((n_items * 32 + 255) / 256), 256, 0, st>>>(offsets, tids, n_items, tids_pad);
    }
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    if (cudaMemcpyAsync(task_d, task.data(), task.size() * sizeof(int2), cudaMemcpyHostToDevice, st) != cudaSuccess) {
        cleanup();
        set_error("merge path: task upload failed");
        return BATMAP_E_CUDA;
    }
    for (int attempt = 0; attempt < 2; ++attempt) {
        dfree(keys, st);
        dfree(vals, st);
        keys = nullptr;
        vals = nullptr;
        if ((rc = dalloc_t(&keys, 2 * kcap, st)) != BATMAP_OK || (rc = dalloc_t(&vals, 2 * kcap, st)) != BATMAP_OK) break;
        cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st);
        cudaEventRecord(e0, st);
        if (stage_b)
            k_merge<true, true><<<(unsigned)task.size(), kMergeThreads, smem, st>>>(
                offsets, tids, tids_pad, cap, items, ns, task_d, cap, threshold, keys, vals, ctr, kcap);
        else
            k_merge<false, false><<<(unsigned)task.size(), kMergeThreads, 0, st>>>(
                offsets, tids, tids_pad, cap, items, ns, task_d, 0, threshold, keys, vals, ctr, kcap);
        cudaEventRecord(e1, st);
        unsigned long long K = 0;
        if (cudaGetLastError() != cudaSuccess ||
            cudaMemcpyAsync(&K, ctr, sizeof(K), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            set_error("merge path: %s", cudaGetErrorString(cudaGetLastError()));
            rc = BATMAP_E_CUDA;
            break;
        }
        if ((int64_t)K > kcap) {
            kcap = (int64_t)K + 1024;
            continue;
        }
        *n_out = (int64_t)K;
        if (kernel_ms) {
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            *kernel_ms = ms;
        }
        if ((int64_t)K > capacity) {
            set_error("capacity %lld < %lld results", (long long)capacity, (long long)K);
            rc = BATMAP_E_CAPACITY;
            break;
        }
        rc = emit_sorted_keys(keys, vals, (int64_t)K, kcap, out, st);
        break;
    }
    cleanup();
    return rc;
}

}  // namespace bm
