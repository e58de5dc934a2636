// util.cu -- errors, allocation, π parameters.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace bm {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

const char* get_error() { return g_err; }

// The device's default memory pool keeps freed blocks instead of returning them to the driver at
// every synchronisation (release threshold 0 by default): a bench step builds and frees GBs of
// BatMaps, and re-mapping them cost ~1 ms per build on C4.  Set once per device per process.
static void keep_pool(cudaStream_t s) {
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return;
    }
    if (done[dev]) return;
    done[dev] = true;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    (void)s;
}

batmap_status dalloc(void** p, size_t bytes, cudaStream_t s) {
    keep_pool(s);
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("cudaMallocAsync(%zu bytes): %s", bytes, cudaGetErrorString(e));
        *p = nullptr;
        return e == cudaErrorMemoryAllocation ? BATMAP_E_NOMEM : BATMAP_E_CUDA;
    }
    return BATMAP_OK;
}

void dfree(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// Per-thread pinned staging for the build's small host <-> device arrays (grown on demand, kept
// for the thread's lifetime).  Copies from / to it are asynchronous; every build synchronises its
// stream (the failure count) before it returns, so the next build of the thread never overwrites
// bytes still in flight.  Returns nullptr (callers fall back to pageable copies) if pinning fails.
batmap_status check_tids_device(const int64_t* offsets, const int32_t* tids, int64_t n_items, cudaStream_t st) {
    if (tids || n_items <= 0) return BATMAP_OK;
    int64_t nnz = 0;
    if (cudaMemcpyAsync(&nnz, offsets + n_items, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("reading offsets[n_items]: %s", cudaGetErrorString(cudaGetLastError()));
        return BATMAP_E_CUDA;
    }
    if (nnz != 0) {
        set_error("tids is NULL but offsets[n_items] = %lld", (long long)nnz);
        return BATMAP_E_INVALID;
    }
    return BATMAP_OK;
}

void* host_staging(size_t bytes, int slot) {
    static thread_local void* buf[2] = {nullptr, nullptr};
    static thread_local size_t cap[2] = {0, 0};
    if (bytes <= cap[slot]) return buf[slot];
    if (buf[slot]) cudaFreeHost(buf[slot]);
    buf[slot] = nullptr;
    cap[slot] = 0;
    size_t want = bytes + bytes / 2 + 4096;
    if (cudaHostAlloc(&buf[slot], want, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        buf[slot] = nullptr;
        return nullptr;
    }
    cap[slot] = want;
    return buf[slot];
}

// Scalar readbacks through a small pinned buffer (one per host thread, allocated once): the
// copies are queued without blocking the host and one stream synchronisation covers them all;
// device -> pageable copies would each block until the stream drains.
batmap_status read_scalars(cudaStream_t st, int k, const void* const* src, const size_t* bytes, void* const* dst) {
    static thread_local uint64_t* pin = nullptr;
    static thread_local bool tried = false;
    if (!tried) {
        tried = true;
        if (cudaHostAlloc(reinterpret_cast<void**>(&pin), 16 * sizeof(uint64_t), cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            pin = nullptr;
        }
    }
    for (int i = 0; i < k; ++i) {
        void* to = pin && k <= 16 && bytes[i] <= 8 ? static_cast<void*>(pin + i) : dst[i];
        BM_CUDA(cudaMemcpyAsync(to, src[i], bytes[i], cudaMemcpyDeviceToHost, st));
    }
    BM_CUDA(cudaStreamSynchronize(st));
    if (pin && k <= 16)
        for (int i = 0; i < k; ++i)
            if (bytes[i] <= 8) memcpy(dst[i], pin + i, bytes[i]);
    return BATMAP_OK;
}

static uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Round keys k_{t,r} = (low32(splitmix64(seed + (4t + r)·φ)) | 1) mod 2^w  (reading #3).
PiParams make_pi(uint64_t seed, int s, const uint32_t* table) {
    PiParams P{};
    P.s = (uint32_t)s;
    P.w = (uint32_t)s + 7u;
    P.U = 127u << s;
    P.mask = (P.w >= 32) ? 0xFFFFFFFFu : ((1u << P.w) - 1u);
    P.half = (P.w + 1u) / 2u;
    for (int t = 0; t < 3; ++t)
        for (int r = 0; r < 4; ++r) {
            uint64_t z = splitmix64(seed + (uint64_t)(4 * t + r) * 0x9E3779B97F4A7C15ull);
            P.key[t][r] = (((uint32_t)z) | 1u) & P.mask;
            uint32_t inv = P.key[t][r];  // Newton: inv <- inv (2 - k inv), 5 steps reach 32 bits
            for (int it = 0; it < 5; ++it) inv *= 2u - P.key[t][r] * inv;
            P.kinv[t][r] = inv & P.mask;
        }
    P.table = table;
    return P;
}

}  // namespace bm
