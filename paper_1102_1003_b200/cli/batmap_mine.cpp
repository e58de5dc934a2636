// batmap_mine -- command-line frequent-pair mining from a FIMI-repository file on one B200, through
// the C ABI only (include/batmap.h): the paper's use case.
//
//   batmap_mine <file.dat> <min_support> [--seed S] [--quiet]
//
// min_support is a transaction count (e.g. 100), or a fraction of the transactions written as a
// percentage ("0.5%") or a number below 1 ("0.005"): s = ceil(fraction * m), at least 1.
//
// Reads the file (one transaction per line, whitespace-separated item labels), parses it on the
// device (batmap_fimi_parse), drops items with support below min_support (batmap_fimi_filter,
// P:118), builds the BatMaps (batmap_build) and emits every pair of items whose support is at
// least min_support (batmap_pair_supports), as "label_i label_j support" lines sorted by
// (label_i, label_j).  Timings and sizes go to stderr.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <cmath>
#include <vector>

#include "batmap.h"

static int fail(const char* what, batmap_status rc) {
    fprintf(stderr, "batmap_mine: %s failed (%d): %s\n", what, (int)rc, batmap_last_error());
    return 1;
}

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            fprintf(stderr, "batmap_mine: %s -> %s\n", #x, cudaGetErrorString(e_));      \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: %s <file.dat> <min_support> [--seed S] [--quiet]\n", argv[0]);
        return 2;
    }
    const char* path = argv[1];
    const char* s_arg = argv[2];
    const size_t s_len = strlen(s_arg);
    const bool percent = s_len > 0 && s_arg[s_len - 1] == '%';
    const double s_val = strtod(s_arg, nullptr);
    const bool relative = percent || (s_val > 0.0 && s_val < 1.0);
    long long s = relative ? 1 : atoll(s_arg);
    uint64_t seed = 0;
    bool quiet = false;
    for (int a = 3; a < argc; ++a) {
        if (!strcmp(argv[a], "--seed") && a + 1 < argc) seed = strtoull(argv[++a], nullptr, 10);
        else if (!strcmp(argv[a], "--quiet")) quiet = true;
    }
    if (!(s_val > 0.0) || (!relative && (s < 1 || s > 0xFFFFFFFFll))) {
        fprintf(stderr, "batmap_mine: min_support must be in [1, 2^32)\n");
        return 2;
    }
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    FILE* f = fopen(path, "rb");
    if (!f) {
        perror(path);
        return 1;
    }
    fseek(f, 0, SEEK_END);
    const long long n_bytes = ftell(f);
    fseek(f, 0, SEEK_SET);
    uint8_t* host = nullptr;
    CK(cudaMallocHost(&host, (size_t)(n_bytes > 0 ? n_bytes : 1)));
    if (n_bytes > 0 && fread(host, 1, (size_t)n_bytes, f) != (size_t)n_bytes) {
        fprintf(stderr, "batmap_mine: short read of %s\n", path);
        return 1;
    }
    fclose(f);
    const auto t1 = now();
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    uint8_t* text = nullptr;
    CK(cudaMalloc(&text, (size_t)(n_bytes > 0 ? n_bytes : 1)));
    CK(cudaMemcpyAsync(text, host, (size_t)n_bytes, cudaMemcpyHostToDevice, st));
    batmap_fimi_handle db = nullptr;
    int64_t bad_line = -1;
    batmap_status rc = batmap_fimi_parse(text, n_bytes, (batmap_stream_t)st, &db, &bad_line);
    if (rc != BATMAP_OK) return fail("parse", rc);
    int64_t n_all = 0, nnz_all = 0, m = 0;
    batmap_fimi_info(db, &n_all, &nnz_all, &m);
    if (relative) {  // a fraction of the transactions (support counts transactions)
        const double frac = percent ? s_val / 100.0 : s_val;
        s = (long long)std::ceil(frac * (double)m - 1e-9);
        if (s < 1) s = 1;
    }
    if ((rc = batmap_fimi_filter(db, (uint32_t)s, (batmap_stream_t)st)) != BATMAP_OK) return fail("filter", rc);
    int64_t n = 0, nnz = 0;
    batmap_fimi_info(db, &n, &nnz, &m);
    int64_t* off = nullptr;
    int32_t* tids = nullptr;
    uint32_t* labels_d = nullptr;
    CK(cudaMalloc(&off, (size_t)(n + 1) * sizeof(int64_t)));
    CK(cudaMalloc(&tids, (size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t)));
    CK(cudaMalloc(&labels_d, (size_t)(n > 0 ? n : 1) * sizeof(uint32_t)));
    if ((rc = batmap_fimi_export(db, off, tids, labels_d, (batmap_stream_t)st)) != BATMAP_OK) return fail("export", rc);
    std::vector<uint32_t> labels((size_t)n);
    if (n) CK(cudaMemcpyAsync(labels.data(), labels_d, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    batmap_fimi_destroy(db);
    cudaFree(text);
    const auto t2 = now();
    std::vector<batmap_triple> out;
    int64_t K = 0;
    if (n >= 2) {
        batmap_build_opts opts;
        memset(&opts, 0, sizeof(opts));
        opts.seed = seed;
        batmap_handle h = nullptr;
        if ((rc = batmap_build(off, tids, n, m > 0 ? m : 1, &opts, (batmap_stream_t)st, &h)) != BATMAP_OK)
            return fail("build", rc);
        batmap_triple* out_d = nullptr;
        int64_t cap = 1 << 20;
        for (int attempt = 0; attempt < 2; ++attempt) {
            CK(cudaMalloc(&out_d, (size_t)cap * sizeof(batmap_triple)));
            rc = batmap_pair_supports(h, nullptr, 0, (uint32_t)s, out_d, cap, &K, (batmap_stream_t)st);
            if (rc != BATMAP_E_CAPACITY) break;
            cudaFree(out_d);
            cap = K;
        }
        if (rc != BATMAP_OK) return fail("pair_supports", rc);
        out.resize((size_t)K);
        if (K) CK(cudaMemcpyAsync(out.data(), out_d, (size_t)K * sizeof(batmap_triple), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cudaFree(out_d);
        batmap_destroy(h);
    }
    const auto t3 = now();
    // dense ids ascend with the labels, so (label_i, label_j) order = (i, j) order
    std::vector<char> buf;
    buf.reserve((size_t)K * 24 + 1);
    char line[64];
    for (const batmap_triple& t : out) {
        const int len = snprintf(line, sizeof(line), "%u %u %u\n", labels[t.i], labels[t.j], t.support);
        buf.insert(buf.end(), line, line + len);
    }
    if (!buf.empty()) fwrite(buf.data(), 1, buf.size(), stdout);
    if (!quiet)
        fprintf(stderr,
                "batmap_mine: %lld bytes, %lld transactions, %lld items (%lld with support >= %lld), %lld pairs with "
                "support >= %lld; read %.1f ms, parse+filter %.1f ms, build+pairs %.1f ms\n",
                n_bytes, (long long)m, (long long)n_all, (long long)n, s, (long long)K, s, ms(t0, t1), ms(t1, t2),
                ms(t2, t3));
    cudaFree(off);
    cudaFree(tids);
    cudaFree(labels_d);
    cudaFreeHost(host);
    cudaStreamDestroy(st);
    return 0;
}
