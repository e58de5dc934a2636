// fimi.h -- the FIMI ingestion handle (ingest.cu, capi.cu).
#pragma once

#include <stdint.h>

struct batmap_fimi {
    int64_t n_items = 0, nnz = 0, m = 0;  // items (distinct labels), (item, tid) pairs, transactions
    int64_t* off_d = nullptr;             // [device] n_items + 1
    int32_t* tids_d = nullptr;            // [device] nnz
    uint32_t* labels_d = nullptr;         // [device] n_items: dense id -> label
};
