// plan.cu -- host-side planner of ★K2: width-class rectangles, 128 x 128 tiles with the
// symmetry cut p <= q, virtualised skinny rectangles, split-K for long tiles, and
// the deal of work to the parts of a multi-GPU run.
#include <algorithm>

#include "plan.h"

namespace bm {

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

void plan_work(const std::vector<ClassInfo>& cls, int part, int n_parts, int grid_cap, bool allow_virtual,
               bool allow_split, Plan* out) {
    Plan& P = *out;
    P = Plan();
    const int C = (int)cls.size();
    // ---- rectangles
    for (int a = 0; a < C; ++a)
        for (int b = a; b < C; ++b) {
            const ClassInfo &A = cls[a], &B = cls[b];
            if (A.n == 0 || B.n == 0 || (a == b && A.n < 2)) continue;
            const int R = B.W / A.W;
            bool virt = false;
            if (allow_virtual && a < b && R > 1) {
                const int64_t normal = ceil_div(B.n, kTile) * kTile * (int64_t)B.W;
                const int64_t vcost = ceil_div((int64_t)B.n * R, kTile) * kTile * (int64_t)A.W;
                virt = vcost * 10 < normal * 7;  // worth a copy + accumulation only if >30% less work
            }
            Rect r{};
            r.cls_a = a;
            r.cls_b = b;
            r.map_a = a;
            r.W_a = A.W;
            r.n_rows = A.n;
            r.row_first = (int32_t)A.first;
            r.col_first = (int32_t)B.first;
            r.diag = (a == b);
            r.n_cols_real = B.n;
            if (virt) {
                VirtCopy vc{};
                vc.cls_b = b;
                vc.W_a = A.W;
                vc.R = R;
                vc.vpad = (int32_t)(ceil_div((int64_t)B.n * R, kTile) * kTile);
                vc.dst_word_off = P.virt_words;
                P.virt_words += (int64_t)A.W * vc.vpad;
                r.map_b = C + (int32_t)P.virt.size();
                P.virt.push_back(vc);
                r.W = A.W;
                r.n_cols = B.n * R;
                r.R = R;
                r.acc = 1;
            } else {
                r.map_b = b;
                r.W = B.W;
                r.n_cols = B.n;
                r.R = 1;
                r.acc = 0;
            }
            P.rects.push_back(r);
        }
    // ---- split-K: tiles far longer than an even share of the work are cut along k
    auto tile_cost = [](const Rect& r) { return (int64_t)kTile * kTile * r.W; };
    int64_t total = 0;
    for (const Rect& r : P.rects) {
        const int64_t ta = ceil_div(r.n_rows, kTile), tb = ceil_div(r.n_cols, kTile);
        const int64_t nt = r.diag ? ta * (ta + 1) / 2 : ta * tb;
        total += nt * tile_cost(r);
    }
    const int64_t target = std::max<int64_t>(1, total / ((int64_t)n_parts * 4 * std::max(grid_cap, 1)));
    if (allow_split)
        for (Rect& r : P.rects)
            if (tile_cost(r) > 2 * target && r.W / kChunk > 1) r.acc = 1;
    // ---- counters of accumulated rectangles
    for (Rect& r : P.rects)
        if (r.acc) {
            r.cnt_off = P.cnt_entries;
            P.cnt_entries += (int64_t)r.n_rows * r.n_cols_real;
        }
    if (P.cnt_entries > (int64_t(1) << 29) && (allow_virtual || allow_split)) {  // > 2 GB of counters
        plan_work(cls, part, n_parts, grid_cap, false, false, out);
        return;
    }
    // ---- units dealt to the parts: a tile row of an accumulated rectangle (all contributions
    // to its pairs stay on one part), or a single tile otherwise
    struct Unit {
        int32_t rect, ti, tj;  // tj = -1: whole tile row
        int64_t cost;
    };
    std::vector<Unit> units;
    for (int ri = 0; ri < (int)P.rects.size(); ++ri) {
        const Rect& r = P.rects[ri];
        const int ta = (int)ceil_div(r.n_rows, kTile), tb = (int)ceil_div(r.n_cols, kTile);
        for (int i = 0; i < ta; ++i) {
            const int j0 = r.diag ? i : 0;
            if (r.acc) {
                units.push_back({ri, i, -1, (int64_t)(tb - j0) * tile_cost(r)});
            } else {
                for (int j = j0; j < tb; ++j) units.push_back({ri, i, j, tile_cost(r)});
            }
        }
    }
    std::stable_sort(units.begin(), units.end(), [](const Unit& x, const Unit& y) { return x.cost > y.cost; });
    struct WorkC {
        Work w;
        int64_t cost;
    };
    std::vector<WorkC> work;
    for (size_t k = 0; k < units.size(); ++k) {
        if ((int)(k % (size_t)n_parts) != part) continue;
        const Unit& u = units[k];
        const Rect& r = P.rects[u.rect];
        const int tb = (int)ceil_div(r.n_cols, kTile);
        const int64_t rows = std::min<int64_t>(kTile, r.n_rows - (int64_t)u.ti * kTile);
        const int W_real = r.W * r.R;
        if (r.acc) P.units.push_back({u.rect, u.ti});
        // algorithmic compares of the pairs this unit owns
        if (r.acc && r.diag) {
            const int64_t r0 = (int64_t)u.ti * kTile;
            for (int64_t q = r0; q < r0 + rows; ++q) P.word_compares += (int64_t)(r.n_rows - 1 - q) * W_real;
        } else if (r.acc) {
            P.word_compares += rows * r.n_cols_real * (int64_t)W_real;
        }
        const int jb = u.tj >= 0 ? u.tj : (r.diag ? u.ti : 0);
        const int je = u.tj >= 0 ? u.tj + 1 : tb;
        for (int j = jb; j < je; ++j) {
            if (!r.acc) {
                const int64_t cols = std::min<int64_t>(kTile, r.n_cols - (int64_t)j * kTile);
                const int64_t pairs = (r.diag && j == u.ti) ? rows * (rows - 1) / 2 : rows * cols;
                P.word_compares += pairs * (int64_t)W_real;
            }
            const int nk = r.W / kChunk;
            int pieces = 1;
            if (r.acc && tile_cost(r) > 2 * target) pieces = (int)std::min<int64_t>(nk, ceil_div(tile_cost(r), target));
            for (int p = 0; p < pieces; ++p) {
                Work w{};
                w.rect = u.rect;
                w.ti = u.ti;
                w.tj = j;
                w.k0 = (int32_t)((int64_t)nk * p / pieces);
                w.k1 = (int32_t)((int64_t)nk * (p + 1) / pieces);
                const int64_t c = (int64_t)(w.k1 - w.k0) * kChunk * kTile * kTile;
                work.push_back({w, c});
                P.tile_compares += c;
            }
        }
    }
    std::stable_sort(work.begin(), work.end(), [](const WorkC& x, const WorkC& y) { return x.cost > y.cost; });
    // ---- the tail of the schedule: the last grid_cap items (the shortest, claimed last) are whole
    // tiles of ordinary rectangles; cut each into pieces along k so that the CTAs finish within a
    // piece of each other (C2: makespan/mean 1.046 -> 1.005 in the planner's cost model).  The
    // pieces write partial counts to their own slices; k2_tail_threshold sums and tests them.
    if (allow_split && grid_cap > 0 && !work.empty()) {
        const size_t n = work.size();
        const size_t begin = n > (size_t)grid_cap ? n - (size_t)grid_cap : 0;
        std::vector<WorkC> pieces;
        int pcs = 0;
        for (size_t k = begin; k < n; ++k) {
            const Work w = work[k].w;
            const Rect& r = P.rects[w.rect];
            const int nk = r.W / kChunk;
            if (pcs == 0) pcs = nk >= 64 ? 8 : (nk >= 16 ? 4 : (nk >= 4 ? 2 : 1));
            if (pcs < 2 || r.acc || w.k0 != 0 || w.k1 != nk || nk < 2 * pcs) continue;
            const int t = (int)P.tails.size();
            P.tails.push_back({w.rect, w.ti, w.tj, 0});
            for (int p = 0; p < pcs; ++p) {
                Work wp = w;
                wp.k0 = (int32_t)((int64_t)nk * p / pcs);
                wp.k1 = (int32_t)((int64_t)nk * (p + 1) / pcs);
                wp.tail = 1 + t * pcs + p;
                const WorkC wc{wp, (int64_t)(wp.k1 - wp.k0) * kChunk * kTile * kTile};
                if (p == 0) work[k] = wc;
                else pieces.push_back(wc);
            }
        }
        if (!P.tails.empty()) {
            P.tail_pieces = pcs;
            work.insert(work.end(), pieces.begin(), pieces.end());
            std::stable_sort(work.begin(), work.end(),
                             [](const WorkC& x, const WorkC& y) { return x.cost > y.cost; });
        }
    }
    P.work.reserve(work.size());
    for (const WorkC& w : work) P.work.push_back(w.w);
}

}  // namespace bm
