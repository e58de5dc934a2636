// dense.cu -- NEXT-1 comparison path: the dense-bitmap formulation of all-pairs support counting
// ("a bitmap to store a vertical representation ... perform the bit-wise AND
// ... and count the number of 1s").  On B200 the AND-and-count of 0/1 bitmaps is the integer
// matrix product X^T X of the m x n incidence matrix, which runs on the tensor cores:
// X is materialised as int8 (one byte per (transaction, item)), C = X^T X is computed by
// cuBLASLt's int8 GEMM (kind::i8 tensor cores, int32 accumulation) in row blocks of the upper
// triangle, and a threshold kernel emits the (i, j, C_ij) with C_ij >= s.  Exact, no failures,
// no corrections.  Not the BatMap method: it is the comparison of SURVEY §8(f) NEXT-1, for the
// dense end of config 5.
#include <cublasLt.h>
#include <dlfcn.h>

#include <algorithm>
#include <cub/cub.cuh>
#include <mutex>

#include "common.cuh"

namespace bm {

namespace {

// cuBLASLt is loaded on first use (no link-time dependency of the BatMap path on it).
struct LtApi {
    bool ok = false;
    cublasLtHandle_t h = nullptr;
    decltype(&cublasLtCreate) create;
    decltype(&cublasLtMatmulDescCreate) descCreate;
    decltype(&cublasLtMatmulDescDestroy) descDestroy;
    decltype(&cublasLtMatmulDescSetAttribute) descSet;
    decltype(&cublasLtMatrixLayoutCreate) layoutCreate;
    decltype(&cublasLtMatrixLayoutDestroy) layoutDestroy;
    decltype(&cublasLtMatmulPreferenceCreate) prefCreate;
    decltype(&cublasLtMatmulPreferenceDestroy) prefDestroy;
    decltype(&cublasLtMatmulPreferenceSetAttribute) prefSet;
    decltype(&cublasLtMatmulAlgoGetHeuristic) heuristic;
    decltype(&cublasLtMatmul) matmul;
};

LtApi& lt() {
    static LtApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* so = dlopen("libcublasLt.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!so) so = dlopen("/usr/local/cuda/lib64/libcublasLt.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!so) return;
#define BM_SYM(field, name)                                          \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(so, name)); \
    if (!api.field) return;
        BM_SYM(create, "cublasLtCreate");
        BM_SYM(descCreate, "cublasLtMatmulDescCreate");
        BM_SYM(descDestroy, "cublasLtMatmulDescDestroy");
        BM_SYM(descSet, "cublasLtMatmulDescSetAttribute");
        BM_SYM(layoutCreate, "cublasLtMatrixLayoutCreate");
        BM_SYM(layoutDestroy, "cublasLtMatrixLayoutDestroy");
        BM_SYM(prefCreate, "cublasLtMatmulPreferenceCreate");
        BM_SYM(prefDestroy, "cublasLtMatmulPreferenceDestroy");
        BM_SYM(prefSet, "cublasLtMatmulPreferenceSetAttribute");
        BM_SYM(heuristic, "cublasLtMatmulAlgoGetHeuristic");
        BM_SYM(matmul, "cublasLtMatmul");
#undef BM_SYM
        if (api.create(&api.h) != CUBLAS_STATUS_SUCCESS) return;
        api.ok = true;
    });
    return api;
}

}  // namespace

// warp per selected item: row r of the item-major bitmap gets a 1 at every tid of S_item
__global__ void k_fill_bitmap(const int64_t* __restrict__ offsets, const int32_t* __restrict__ tids,
                              const int32_t* __restrict__ sel, int64_t n_sel, int64_t m_pad, int8_t* __restrict__ X) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (r >= n_sel) return;
    const int32_t item = sel ? sel[r] : (int32_t)r;
    int8_t* row = X + r * m_pad;
    for (int64_t k = offsets[item] + lane; k < offsets[item + 1]; k += 32) row[tids[k]] = 1;
}

// C is the column-major (rows x cols) block of X^T X for selection rows [r0, r0 + rows) and
// columns [r0, r0 + cols): emit (i, j, C) for i < j, C >= thr.
__global__ void k_dense_threshold(const int32_t* __restrict__ C, int64_t r0, int64_t rows, int64_t cols, int64_t n_sel,
                                  const int32_t* __restrict__ sel, uint32_t thr, uint64_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals, unsigned long long* __restrict__ ctr, int64_t cap) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * cols) return;
    const int64_t jl = e / rows, il = e - jl * rows;
    const int64_t i = r0 + il, j = r0 + jl;
    if (i >= n_sel || j >= n_sel || j <= i) return;
    const uint32_t c = (uint32_t)C[e];
    if (c < thr) return;
    uint32_t a = (uint32_t)(sel ? sel[i] : i), b = (uint32_t)(sel ? sel[j] : j);
    if (a > b) {
        const uint32_t t = a;
        a = b;
        b = t;
    }
    const unsigned long long at = atomicAdd(ctr, 1ull);
    if ((int64_t)at < cap) {
        keys[at] = ((uint64_t)a << 32) | b;
        vals[at] = c;
    }
}

__global__ void k_dense_emit(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                             batmap_triple* __restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    batmap_triple t;
    t.i = (uint32_t)(keys[k] >> 32);
    t.j = (uint32_t)keys[k];
    t.support = vals[k];
    out[k] = t;
}

static batmap_status lt_check(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) {
        set_error("cuBLASLt %s failed (status %d)", what, (int)s);
        return BATMAP_E_CUDA;
    }
    return BATMAP_OK;
}

// C (rows x cols, col-major, ld rows) = A^T B with A = X[:, rows block] (m_pad x rows, ld m_pad),
// B = X[:, cols block] (m_pad x cols, ld m_pad): int8 inputs, int32 accumulate (TN layout).
static batmap_status gemm_int8(const int8_t* A, const int8_t* B, int32_t* C, int64_t rows, int64_t cols, int64_t m_pad,
                               void* ws, size_t ws_bytes, cudaStream_t st) {
    LtApi& L = lt();
    cublasLtMatmulDesc_t desc = nullptr;
    cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
    cublasLtMatmulPreference_t pref = nullptr;
    batmap_status rc = BATMAP_OK;
    const int32_t alpha = 1, beta = 0;
    const cublasOperation_t opT = CUBLAS_OP_T, opN = CUBLAS_OP_N;
    do {
        if ((rc = lt_check(L.descCreate(&desc, CUBLAS_COMPUTE_32I, CUDA_R_32I), "desc")) != BATMAP_OK) break;
        if ((rc = lt_check(L.descSet(desc, CUBLASLT_MATMUL_DESC_TRANSA, &opT, sizeof(opT)), "transa")) != BATMAP_OK) break;
        if ((rc = lt_check(L.descSet(desc, CUBLASLT_MATMUL_DESC_TRANSB, &opN, sizeof(opN)), "transb")) != BATMAP_OK) break;
        if ((rc = lt_check(L.layoutCreate(&la, CUDA_R_8I, m_pad, rows, m_pad), "layout A")) != BATMAP_OK) break;
        if ((rc = lt_check(L.layoutCreate(&lb, CUDA_R_8I, m_pad, cols, m_pad), "layout B")) != BATMAP_OK) break;
        if ((rc = lt_check(L.layoutCreate(&lc, CUDA_R_32I, rows, cols, rows), "layout C")) != BATMAP_OK) break;
        if ((rc = lt_check(L.prefCreate(&pref), "pref")) != BATMAP_OK) break;
        uint64_t wsb = ws_bytes;
        if ((rc = lt_check(L.prefSet(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb)), "pref ws")) !=
            BATMAP_OK)
            break;
        cublasLtMatmulHeuristicResult_t res{};
        int n_res = 0;
        if ((rc = lt_check(L.heuristic(L.h, desc, la, lb, lc, lc, pref, 1, &res, &n_res), "heuristic")) != BATMAP_OK)
            break;
        if (n_res == 0) {
            set_error("cuBLASLt: no int8 algorithm for %lld x %lld x %lld", (long long)rows, (long long)cols,
                      (long long)m_pad);
            rc = BATMAP_E_CUDA;
            break;
        }
        rc = lt_check(L.matmul(L.h, desc, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &res.algo, ws, ws_bytes, st),
                      "matmul");
    } while (0);
    if (pref) L.prefDestroy(pref);
    if (lc) L.layoutDestroy(lc);
    if (lb) L.layoutDestroy(lb);
    if (la) L.layoutDestroy(la);
    if (desc) L.descDestroy(desc);
    return rc;
}

// (key = i << 32 | j, value = support) pairs in keys[0, K) / vals[0, K) (each buffer 2 cap long:
// the radix sort's double buffer) -> out[0, K) sorted by (i, j); synchronises st.
batmap_status emit_sorted_keys(uint64_t* keys, uint32_t* vals, int64_t K, int64_t cap, batmap_triple* out,
                               cudaStream_t st) {
    if (K > 1) {
        cub::DoubleBuffer<uint64_t> dk(keys, keys + cap);
        cub::DoubleBuffer<uint32_t> dv(vals, vals + cap);
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)K, 0, 64, st);
        void* tmp = nullptr;
        BM_TRY(dalloc(&tmp, tb + 16, st));
        cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)K, 0, 64, st);
        k_dense_emit<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(dk.Current(), dv.Current(), K, out);
        dfree(tmp, st);
    } else if (K == 1) {
        k_dense_emit<<<1, 32, 0, st>>>(keys, vals, 1, out);
    }
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("sort/emit of the result: %s", cudaGetErrorString(cudaGetLastError()));
        return BATMAP_E_CUDA;
    }
    return BATMAP_OK;
}

batmap_status dense_pair_supports(const int64_t* offsets, const int32_t* tids, int64_t n_items, int64_t m,
                                  const int32_t* items, int64_t n_sel, uint32_t threshold, batmap_triple* out,
                                  int64_t capacity, int64_t* n_out, double* gemm_ms, cudaStream_t st) {
    LtApi& L = lt();
    if (!L.ok) {
        set_error("cuBLASLt could not be loaded (libcublasLt.so.12)");
        return BATMAP_E_CUDA;
    }
    const int64_t ns = items ? n_sel : n_items;
    *n_out = 0;
    if (gemm_ms) *gemm_ms = 0;
    if (ns < 2) return BATMAP_OK;
    const int64_t m_pad = (m + 127) / 128 * 128;
    const int64_t n_pad = (ns + 127) / 128 * 128;
    if ((double)m_pad * n_pad > 48e9) {
        set_error("dense bitmap of %lld x %lld bytes exceeds the 48 GB budget", (long long)n_pad, (long long)m_pad);
        return BATMAP_E_NOMEM;
    }
    // row block so that one int32 block of C stays under 512 MB
    int64_t B = std::max<int64_t>(128, ((int64_t)(512ll << 20) / (4 * n_pad)) / 128 * 128);
    B = std::min(B, n_pad);
    int8_t* X = nullptr;
    int32_t* C = nullptr;
    void* ws = nullptr;
    const size_t ws_bytes = 64ull << 20;
    uint64_t* keys = nullptr;
    uint32_t* vals = nullptr;
    unsigned long long* ctr = nullptr;
    int64_t cap = std::max<int64_t>(1 << 20, 16 * ns);
    batmap_status rc = BATMAP_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto cleanup = [&]() {
        dfree(X, st);
        dfree(C, st);
        dfree(ws, st);
        dfree(keys, st);
        dfree(vals, st);
        dfree(ctr, st);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    };
    if ((rc = dalloc_t(&X, n_pad * m_pad, st)) != BATMAP_OK || (rc = dalloc_t(&C, B * n_pad, st)) != BATMAP_OK ||
        (rc = dalloc(&ws, ws_bytes, st)) != BATMAP_OK || (rc = dalloc_t(&ctr, 1, st)) != BATMAP_OK) {
        cleanup();
        return rc;
    }
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    if (cudaMemsetAsync(X, 0, (size_t)(n_pad * m_pad), st) != cudaSuccess) {
        cleanup();
        set_error("memset failed");
        return BATMAP_E_CUDA;
    }
    k_fill_bitmap<<<(unsigned)((ns * 32 + 255) / 256), 256, 0, st>>>(offsets, tids, items, ns, m_pad, X);
    for (int attempt = 0; attempt < 2; ++attempt) {
        dfree(keys, st);
        dfree(vals, st);
        keys = nullptr;
        vals = nullptr;
        if ((rc = dalloc_t(&keys, 2 * cap, st)) != BATMAP_OK || (rc = dalloc_t(&vals, 2 * cap, st)) != BATMAP_OK) break;
        cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st);
        cudaEventRecord(e0, st);
        for (int64_t r0 = 0; r0 < ns && rc == BATMAP_OK; r0 += B) {
            const int64_t rows = std::min(B, n_pad - r0);
            const int64_t cols = n_pad - r0;  // upper triangle: columns j >= r0
            rc = gemm_int8(X + r0 * m_pad, X + r0 * m_pad, C, rows, cols, m_pad, ws, ws_bytes, st);
            if (rc != BATMAP_OK) break;
            const int64_t cnt = rows * cols;
            k_dense_threshold<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(C, r0, rows, cols, ns, items, threshold,
                                                                             keys, vals, ctr, cap);
        }
        cudaEventRecord(e1, st);
        if (rc != BATMAP_OK) break;
        unsigned long long K = 0;
        if (cudaMemcpyAsync(&K, ctr, sizeof(K), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            set_error("dense path: %s", cudaGetErrorString(cudaGetLastError()));
            rc = BATMAP_E_CUDA;
            break;
        }
        if ((int64_t)K > cap) {
            cap = (int64_t)K + 1024;
            continue;
        }
        *n_out = (int64_t)K;
        if (gemm_ms) {
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            *gemm_ms = ms;
        }
        if ((int64_t)K > capacity) {
            set_error("capacity %lld < %lld results", (long long)capacity, (long long)K);
            rc = BATMAP_E_CAPACITY;
            break;
        }
        rc = emit_sorted_keys(keys, vals, (int64_t)K, cap, out, st);
        break;
    }
    cleanup();
    return rc;
}

}  // namespace bm
