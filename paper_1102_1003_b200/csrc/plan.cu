// plan.cu -- host-side planner of ★K2: width-class rectangles, 128 x tn tiles with the
// symmetry cut p <= q, virtualised skinny rectangles, split-K for long tiles, and
// the deal of work to the parts of a multi-GPU run, and promotion of small narrow classes.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <new>
#include <unordered_map>

#include "plan.h"

namespace bm {

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

namespace {
struct PoolBlock {
    void* p;
    size_t bytes;
    bool busy;
};
std::mutex g_pool_mu;
std::vector<PoolBlock> g_pool;
constexpr size_t kPoolMinBytes = size_t(1) << 20;
constexpr size_t kPoolMaxBlocks = 8;
}  // namespace

void* plan_pool_alloc(size_t bytes) {
    if (bytes < kPoolMinBytes) return ::operator new(bytes);
    std::lock_guard<std::mutex> lk(g_pool_mu);
    PoolBlock* best = nullptr;  // the smallest idle block that fits without hogging a much larger one
    for (PoolBlock& b : g_pool)
        if (!b.busy && b.bytes >= bytes && b.bytes <= 4 * bytes && (!best || b.bytes < best->bytes)) best = &b;
    if (best) {
        best->busy = true;
        return best->p;
    }
    const size_t want = (bytes + kPoolMinBytes - 1) / kPoolMinBytes * kPoolMinBytes;
    void* p = ::operator new(want);
    if (g_pool.size() >= kPoolMaxBlocks) {  // replace the smallest idle block, else do not pool this one
        PoolBlock* victim = nullptr;
        for (PoolBlock& b : g_pool)
            if (!b.busy && (!victim || b.bytes < victim->bytes)) victim = &b;
        if (!victim) return p;  // freed by plan_pool_free's fallback
        ::operator delete(victim->p);
        *victim = PoolBlock{p, want, true};
        return p;
    }
    g_pool.push_back(PoolBlock{p, want, true});
    return p;
}

void plan_pool_free(void* p) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (PoolBlock& b : g_pool)
            if (b.p == p) {
                b.busy = false;
                return;
            }
    }
    ::operator delete(p);
}

// Stable sort by descending cost.  Work lists have few distinct costs (one per rectangle, per
// accumulated tile row or per k-piece length), so this buckets in O(T) instead of comparing
// (C4: 3e5 tiles; the plan is built on the host while the build kernels run).
template <typename V, typename Cost>
static void stable_sort_desc(V& v, Cost cost) {
    std::unordered_map<int64_t, int32_t> first_seen;  // cost -> id in order of first appearance
    std::vector<int64_t> keys;
    std::vector<int32_t> bucket(v.size());
    int64_t last = -1;
    int32_t last_id = -1;
    for (size_t e = 0; e < v.size(); ++e) {
        const int64_t c = cost(v[e]);
        if (c != last) {  // runs of equal cost are the common case
            auto it = first_seen.find(c);  // find first: emplace would allocate a node every time
            if (it == first_seen.end()) {
                it = first_seen.emplace(c, (int32_t)keys.size()).first;
                keys.push_back(c);
            }
            last = c;
            last_id = it->second;
        }
        bucket[e] = last_id;
    }
    std::vector<int32_t> order(keys.size()), rank(keys.size());
    for (size_t k = 0; k < keys.size(); ++k) order[k] = (int32_t)k;
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return keys[a] > keys[b]; });
    for (size_t k = 0; k < order.size(); ++k) rank[order[k]] = (int32_t)k;
    std::vector<int64_t> at(keys.size() + 1, 0);
    for (size_t e = 0; e < v.size(); ++e) ++at[rank[bucket[e]] + 1];
    for (size_t k = 1; k < at.size(); ++k) at[k] += at[k - 1];
    V out(v.size());
    for (size_t e = 0; e < v.size(); ++e) out[at[rank[bucket[e]]]++] = v[e];
    v.swap(out);
}

int lg_ratio(int64_t W, int64_t W_min) {
    if (W_min <= 0 || W < W_min || W % W_min) return -1;
    const int64_t q = W / W_min;
    int l = 0;
    while ((int64_t(1) << l) < q) ++l;
    return (int64_t(1) << l) == q ? l : -1;
}

// Estimated executed compares of tiling classes (n[a], W[a]) the way plan_work does (skinny
// rectangles virtualised when that saves > 30 %), plus the copy traffic of promoted groups
// (a written word ~ 12 compare-equivalents: 4 B at ~1/3 of R_int's compare rate per byte).
// Tiles (ti, tj) of the triangle of n items with 128-row and tn-column tiles that hold a pair i < j:
// tj >= ti * 128 / tn.
static int64_t diag_tiles(int64_t n, int tn) {
    const int64_t ta = ceil_div(n, kTile), tb = ceil_div(n, tn), q = kTile / tn;
    return ta * tb - q * ta * (ta - 1) / 2;
}

static int64_t est_cost(const std::vector<int64_t>& n, const std::vector<int64_t>& W,
                        const std::vector<int64_t>& copy_words, bool allow_virtual, int tn) {
    const int C = (int)n.size();
    const int64_t T2 = (int64_t)kTile * tn;
    int64_t tot = 0;
    for (int a = 0; a < C; ++a) {
        tot += 12 * copy_words[a];
        if (n[a] == 0) continue;
        const int64_t ta = ceil_div(n[a], kTile);
        for (int b = a; b < C; ++b) {
            if (n[b] == 0) continue;
            if (a == b) {
                if (n[a] >= 2) tot += diag_tiles(n[a], tn) * T2 * W[a];
                continue;
            }
            int64_t c = ta * ceil_div(n[b], tn) * T2 * W[b];
            const int64_t R = W[b] / W[a];
            if (allow_virtual && R > 1) {
                const int64_t v = ta * ceil_div(n[b] * R, tn) * T2 * W[a];
                if (v * 10 < c * 7) c = v;
            }
            tot += c;
        }
    }
    return tot;
}

// Greedy promotion: repeatedly merge the adjacent pair of class groups whose merge lowers the
// estimated cost most, while that gains > 1 %.  Groups are runs [lo, hi] of the width-sorted
// classes; a group is planned at its widest member's width.
static std::vector<std::pair<int, int>> choose_groups(const std::vector<ClassInfo>& cls, bool allow_virtual,
                                                      int tn, int64_t* cost_out = nullptr) {
    const int C = (int)cls.size();
    std::vector<std::pair<int, int>> g;
    for (int a = 0; a < C; ++a) g.push_back({a, a});
    auto cost = [&](const std::vector<std::pair<int, int>>& gs) {
        std::vector<int64_t> n, W, cw;
        for (const auto& p : gs) {
            int64_t s = 0;
            for (int a = p.first; a <= p.second; ++a) s += cls[a].n;
            n.push_back(s);
            W.push_back(cls[p.second].W);
            cw.push_back(p.first == p.second ? 0 : ceil_div(s, kPadItems) * kPadItems * cls[p.second].W);
        }
        return est_cost(n, W, cw, allow_virtual, tn);
    };
    bool mergeable = C >= 2;
    for (int a = 0; a < C; ++a)
        if (lg_ratio(cls[a].W, cls[0].W) < 0) mergeable = false;  // widths must be W_0 times powers of two
    if (!mergeable) {
        if (cost_out) *cost_out = cost(g);
        return g;
    }
    constexpr int64_t kMaxPromoWords = int64_t(1) << 27;  // 512 MB per promoted block
    int64_t best = cost(g);
    for (;;) {
        int pick = -1;
        int64_t pick_cost = 0;
        for (size_t k = 0; k + 1 < g.size(); ++k) {
            int64_t s = 0;
            for (int a = g[k].first; a <= g[k + 1].second; ++a) s += cls[a].n;
            if (ceil_div(s, kPadItems) * kPadItems * cls[g[k + 1].second].W > kMaxPromoWords) continue;
            std::vector<std::pair<int, int>> t = g;
            t[k].second = t[k + 1].second;
            t.erase(t.begin() + (long)k + 1);
            const int64_t c = cost(t);
            if (pick < 0 || c < pick_cost) {
                pick = (int)k;
                pick_cost = c;
            }
        }
        if (pick < 0 || pick_cost * 100 >= best * 99) break;
        g[pick].second = g[pick + 1].second;
        g.erase(g.begin() + pick + 1);
        best = pick_cost;
    }
    if (cost_out) *cost_out = best;
    return g;
}

int64_t plan_cost(const std::vector<ClassInfo>& cls, bool allow_virtual, bool allow_promote, int tn) {
    int64_t c = 0;
    if (allow_promote) {
        choose_groups(cls, allow_virtual, tn, &c);
        return c;
    }
    std::vector<int64_t> n, W, cw;
    for (const ClassInfo& k : cls) {
        n.push_back(k.n);
        W.push_back(k.W);
        cw.push_back(0);
    }
    return est_cost(n, W, cw, allow_virtual, tn);
}

// Tile rows per band of the grouped tile order: a band of row tiles of ~32 MB stays in L2 while the
// columns stream past it; rectangles whose operands fit in L2 together (<= 96 MB) stay row-major,
// which re-reads least (measured K2 DRAM reads, profiles/r2_k2_order_dram.json: C4 G = 1 / 2 / 4 /
// 10 / 20 / 40: 988 / 697 / 432 / 227 / 293 / 684 GB; C2 G = 1 / 4 / 8 / 16 / 42: 130 / 133 / 138 /
// 146 / 152 MB; K2 time unchanged within 0.1 % in every case).  BATMAP_K2_GROUP=<rows> overrides.
static int group_rows(const Rect& r, int ta) {
    const char* e = getenv("BATMAP_K2_GROUP");  // once per rectangle
    const int env = e ? atoi(e) : 0;
    if (env > 0) return std::min(env, std::max(ta, 1));
    const int64_t op_bytes = 4ll * ((int64_t)r.n_rows * r.W_a + (r.diag ? 0 : (int64_t)r.n_cols * r.W));
    if (op_bytes <= (int64_t(96) << 20)) return 1;
    const int64_t row_bytes = (int64_t)kTile * r.W_a * 4;
    const int64_t g = (int64_t(32) << 20) / std::max<int64_t>(row_bytes, 1);
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, std::max(ta, 1)));
}

void plan_work(const std::vector<ClassInfo>& orig, int part, int n_parts, int grid_cap, bool allow_virtual,
               bool allow_split, bool allow_promote, Plan* out, int tn) {
    Plan& P = *out;
    P = Plan();
    const int TN = (tn == 64) ? 64 : kTile;  // tile width
    const int QD = kTile / TN;               // tile columns per tile-row step on the diagonal
    P.tn = TN;
    // ---- planned classes: original classes, or promoted groups of adjacent ones
    const std::vector<std::pair<int, int>> groups =
        allow_promote ? choose_groups(orig, allow_virtual, TN) : [&] {
            std::vector<std::pair<int, int>> g;
            for (int a = 0; a < (int)orig.size(); ++a) g.push_back({a, a});
            return g;
        }();
    P.eff_of.assign(orig.size(), -1);
    for (const auto& gr : groups) {
        const int e = (int)P.eff.size();
        for (int a = gr.first; a <= gr.second; ++a) P.eff_of[a] = e;
        if (gr.first == gr.second) {
            P.eff.push_back(orig[gr.first]);
            P.eff_promo.push_back(-1);
            continue;
        }
        ClassInfo c = orig[gr.second];
        c.first = orig[gr.first].first;
        int64_t n = 0;
        for (int a = gr.first; a <= gr.second; ++a) n += orig[a].n;
        c.n = (int32_t)n;
        c.n_pad = (int32_t)(ceil_div(n, kPadItems) * kPadItems);
        c.word_off = P.promo_words;
        PromoCopy pc{};
        pc.cls_lo = gr.first;
        pc.cls_hi = gr.second;
        pc.W = c.W;
        pc.n = c.n;
        pc.n_pad = c.n_pad;
        pc.dst_word_off = P.promo_words;
        P.promo_words += (int64_t)c.n_pad * c.W;
        P.eff_promo.push_back((int32_t)P.promo.size());
        P.promo.push_back(pc);
        P.eff.push_back(c);
    }
    const std::vector<ClassInfo>& cls = P.eff;
    const int C = (int)cls.size();
    const int64_t W_min = orig.empty() ? 1 : orig[0].W;
    // sum of the original widths of planned-class items [q0, q1) (local indices)
    auto sumW = [&](int c, int64_t q0, int64_t q1) -> int64_t {
        if (q1 <= q0) return 0;
        if (P.eff_promo[c] < 0) return (q1 - q0) * cls[c].W;
        const PromoCopy& pc = P.promo[P.eff_promo[c]];
        int64_t s = 0, base = 0;
        for (int a = pc.cls_lo; a <= pc.cls_hi; ++a) {
            const int64_t lo = std::max(q0, base), hi = std::min(q1, base + orig[a].n);
            if (hi > lo) s += (hi - lo) * orig[a].W;
            base += orig[a].n;
        }
        return s;
    };
    // ---- rectangles
    for (int a = 0; a < C; ++a)
        for (int b = a; b < C; ++b) {
            const ClassInfo &A = cls[a], &B = cls[b];
            if (A.n == 0 || B.n == 0 || (a == b && A.n < 2)) continue;
            const int R = B.W / A.W;
            bool virt = false;
            if (allow_virtual && a < b && R > 1) {
                const int64_t normal = ceil_div(B.n, TN) * TN * (int64_t)B.W;
                const int64_t vcost = ceil_div((int64_t)B.n * R, TN) * TN * (int64_t)A.W;
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
            r.promo = P.eff_promo[b] >= 0;
            r.lgK = lg_ratio(B.W, W_min);
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
    auto tile_cost = [&](const Rect& r) { return (int64_t)kTile * TN * r.W; };
    int64_t total = 0;
    for (const Rect& r : P.rects) {
        const int64_t ta = ceil_div(r.n_rows, kTile), tb = ceil_div(r.n_cols, TN);
        const int64_t nt = r.diag ? diag_tiles(r.n_rows, TN) : ta * tb;
        total += nt * tile_cost(r);
    }
    // The split decisions shape the units dealt to the parts, so with n_parts > 1 they use a grid
    // every rank agrees on (a B200's 2 CTAs x 148 SMs), not the local device's: ranks on devices
    // with different SM counts (MIG slices, mixed GPUs) must build identical unit lists, or pairs
    // would be dropped or emitted twice.  grid_cap stays in use for the part-local tail split below.
    const int split_grid = n_parts > 1 ? kDealGrid : std::max(grid_cap, 1);
    const char* fe = getenv("BATMAP_K2_SPLITF");  // split granularity f (measured: 4; test hook)
    const int64_t split_f = fe && atoi(fe) > 0 ? atoi(fe) : 4;
    const int64_t target = std::max<int64_t>(1, total / ((int64_t)n_parts * split_f * split_grid));
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
        const std::vector<ClassInfo> o = orig;
        plan_work(o, part, n_parts, grid_cap, false, false, false, out, tn);
        return;
    }
    // ---- units dealt to the parts: a tile row of an accumulated rectangle (all contributions
    // to its pairs stay on one part), or a single tile otherwise.  Units are ordered by cost,
    // longest first, stable in creation order (rectangle, row, column), and dealt round-robin.
    // They are kept as segments -- all tiles of an ordinary rectangle (equal cost, contiguous in
    // creation order), or one accumulated tile row -- so a part touches only its own 1/n_parts of
    // the units (C4: 3e5 tiles).
    struct Unit {
        int32_t rect, ti, tj;  // tj = -1: whole tile row
        int64_t cost;
    };
    struct Seg {
        int32_t rect, ti;  // ti: the accumulated tile row, or -1 for all tiles of an ordinary rectangle
        int64_t count, cost;
    };
    std::vector<Seg> segs;
    for (int ri = 0; ri < (int)P.rects.size(); ++ri) {
        const Rect& r = P.rects[ri];
        const int ta = (int)ceil_div(r.n_rows, kTile), tb = (int)ceil_div(r.n_cols, TN);
        if (r.acc) {
            for (int i = 0; i < ta; ++i) segs.push_back({ri, i, 1, (int64_t)(tb - (r.diag ? i * QD : 0)) * tile_cost(r)});
        } else {
            const int64_t nt = r.diag ? diag_tiles(r.n_rows, TN) : (int64_t)ta * tb;
            if (nt) segs.push_back({ri, -1, nt, tile_cost(r)});
        }
    }
    stable_sort_desc(segs, [](const Seg& x) { return x.cost; });
    // Work items are emitted in deal order.  The tiles of ordinary rectangles come out already in
    // descending cost order (segments are sorted by their tile cost) and go straight into the
    // reserved list; the k-pieces of accumulated tile rows (few) are generated first, into a side
    // list with their deal position, stably sorted by cost and merged in as the main items are
    // emitted -- the stable descending sort of the deal order without sorting or moving the 3e5
    // items of C4 (a merge from the back afterwards moved every item: 1.5 ms of C4's plan).
    struct Side {
        Work w;
        int64_t cost, pos;  // pos: main items dealt before it
    };
    std::vector<Side> side;
    side.reserve(4096);
    WorkList& items = P.work;
    {  // capacity: this part's share of the tiles, split tiles counted per piece
        int64_t cnt = 0;
        for (const Rect& r : P.rects) {
            const int64_t ta = ceil_div(r.n_rows, kTile), tb = ceil_div(r.n_cols, TN);
            const int64_t nt = r.diag ? diag_tiles(r.n_rows, TN) : ta * tb;
            const int64_t nk = r.W / kChunk;
            const int64_t pieces = (r.acc && tile_cost(r) > 2 * target) ? std::min(nk, ceil_div(tile_cost(r), target)) : 1;
            cnt += nt * pieces;
        }
        items.reserve((size_t)(cnt / n_parts + 8 * 1024));
    }
    // main items go through put(): side items that sort before it (higher cost, or equal cost and
    // dealt no later) are placed first
    size_t si = 0;
    int64_t main_count = 0, main_before = 0;  // main_before: the side pre-pass's deal position
    auto put = [&](const Work& w, int64_t c) {
        while (si < side.size() && (side[si].cost > c || (side[si].cost == c && side[si].pos <= main_count)))
            items.push_back(side[si++].w);
        items.push_back(w);
        ++main_count;
    };
    // one unit of this part, in deal order: its algorithmic compares and its work items
    auto emit = [&](const Unit& u) {
        const Rect& r = P.rects[u.rect];
        const int tb = (int)ceil_div(r.n_cols, TN);
        const int64_t rows = std::min<int64_t>(kTile, r.n_rows - (int64_t)u.ti * kTile);
        const int W_real = r.W * r.R;
        const bool plain_w = P.eff_promo[r.cls_b] < 0;  // every column item has width W_real
        if (r.acc) P.units.push_back({u.rect, u.ti});
        // algorithmic compares of the pairs this unit owns: sum of max(W_i, W_j) = W_j (columns are
        // never narrower than rows: width-sorted positions)
        const int64_t r0 = (int64_t)u.ti * kTile;
        if (r.acc && r.diag) {
            if (plain_w) {
                const int64_t a = r.n_rows - 1 - r0, b = r.n_rows - r0 - rows;  // sum_{q} (n-1-q), q in [r0, r0+rows)
                P.word_compares += (a + b) * rows / 2 * W_real;
            } else {
                for (int64_t q = r0; q < r0 + rows; ++q) P.word_compares += sumW(r.cls_b, q + 1, r.n_rows);
            }
        } else if (r.acc) {
            P.word_compares += rows * sumW(r.cls_b, 0, r.n_cols_real);
        }
        const int jb = u.tj >= 0 ? u.tj : (r.diag ? u.ti * QD : 0);
        const int je = u.tj >= 0 ? u.tj + 1 : tb;
        const int nk = r.W / kChunk;
        int pieces = 1;
        if (r.acc && tile_cost(r) > 2 * target) pieces = (int)std::min<int64_t>(nk, ceil_div(tile_cost(r), target));
        for (int j = jb; j < je; ++j) {
            if (!r.acc) {
                const int64_t c0 = (int64_t)j * TN, c1 = std::min<int64_t>(r.n_cols, c0 + TN);
                if (r.diag && c0 < r0 + rows) {  // the tile straddles the diagonal: pairs q < col only
                    for (int64_t q = r0; q < r0 + rows; ++q) P.word_compares += sumW(r.cls_b, std::max(q + 1, c0), c1);
                } else {
                    P.word_compares += plain_w ? rows * (c1 - c0) * W_real : rows * sumW(r.cls_b, c0, c1);
                }
            }
            for (int p = 0; p < pieces; ++p) {
                Work w{};
                w.rect = u.rect;
                w.ti = u.ti;
                w.tj = j;
                w.k0 = (int32_t)((int64_t)nk * p / pieces);
                w.k1 = (int32_t)((int64_t)nk * (p + 1) / pieces);
                const int64_t c = (int64_t)(w.k1 - w.k0) * kChunk * kTile * TN;
                if (r.acc) side.push_back({w, c, main_before});
                else put(w, c);
                P.tile_compares += c;
            }
        }
    };
    {  // pre-pass: the accumulated tile rows of this part (their k-pieces form the side list)
        int64_t at = 0;
        for (const Seg& g : segs) {
            const int64_t t0 = (((int64_t)part - at) % n_parts + n_parts) % n_parts;
            if (g.ti >= 0) {
                if (t0 == 0) emit(Unit{g.rect, g.ti, -1, g.cost});
            } else if (t0 < g.count) {
                main_before += (g.count - t0 + n_parts - 1) / n_parts;
            }
            at += g.count;
        }
        std::stable_sort(side.begin(), side.end(), [](const Side& x, const Side& y) { return x.cost > y.cost; });
    }
    {
        int64_t at = 0;  // global index of the segment's first unit
        for (const Seg& g : segs) {
            const int64_t t0 = (((int64_t)part - at) % n_parts + n_parts) % n_parts;
            if (g.ti >= 0) {
                // emitted by the pre-pass
            } else if (t0 < g.count) {
                const Rect& r = P.rects[g.rect];
                const int ta = (int)ceil_div(r.n_rows, kTile), tb = (int)ceil_div(r.n_cols, TN);
                // Tiles in grouped order: bands of G tile rows, column by column inside a band, so
                // the CTAs running at once share a band of row tiles (kept in L2) and each column
                // tile is fetched from HBM once per band instead of once per tile row (C4: the
                // 2.4 GB class would otherwise stream ~780 / 2 times).  G = 1 is row-major.
                const int G = group_rows(r, ta);
                if (n_parts == 1) {  // every tile is this part's: closed-form compares, bare items
                    const bool plain_w = P.eff_promo[r.cls_b] < 0;
                    if (r.diag) {
                        const int64_t n = r.n_rows;
                        if (plain_w) P.word_compares += n * (n - 1) / 2 * r.W;
                        else
                            for (int64_t q = 0; q + 1 < n; ++q) P.word_compares += sumW(r.cls_b, q + 1, n);
                    } else {
                        P.word_compares += (int64_t)r.n_rows * (plain_w ? (int64_t)r.n_cols * r.W : sumW(r.cls_b, 0, r.n_cols));
                    }
                    const int nk = r.W / kChunk;
                    const int64_t c = (int64_t)nk * kChunk * kTile * TN;
                    P.tile_compares += g.count * c;
                    while (si < side.size() && side[si].cost > c) items.push_back(side[si++].w);
                    // side items of equal cost land inside the segment, before the main item
                    // whose index reaches their deal position; the rest is one contiguous run
                    size_t ties = 0;
                    while (si + ties < side.size() && side[si + ties].cost == c &&
                           side[si + ties].pos < main_count + g.count)
                        ++ties;
                    const size_t base = items.size();
                    items.resize(base + (size_t)g.count + ties);
                    Work* o = items.data() + base;
                    const size_t tie_end = si + ties;
                    int64_t next_tie = si < tie_end ? side[si].pos : INT64_MAX;
                    for (int i0 = 0; i0 < ta; i0 += G) {
                        const int i1 = std::min(ta, i0 + G);
                        for (int j = r.diag ? i0 * QD : 0; j < tb; ++j) {
                            const int ie = r.diag ? std::min(i1, j / QD + 1) : i1;
                            for (int i = i0; i < ie; ++i) {
                                while (main_count >= next_tie) {
                                    *o++ = side[si++].w;
                                    next_tie = si < tie_end ? side[si].pos : INT64_MAX;
                                }
                                *o++ = Work{g.rect, i, j, 0, nk, 0};
                                ++main_count;
                            }
                        }
                    }
                    at += g.count;
                    continue;
                }
                int64_t t = 0, next = t0;  // unit index at the start of band i0; next unit of this part
                for (int i0 = 0; i0 < ta && next < g.count; i0 += G) {
                    const int i1 = std::min(ta, i0 + G);
                    int64_t band_n = 0;
                    for (int i = i0; i < i1; ++i) band_n += tb - (r.diag ? i * QD : 0);
                    if (next >= t + band_n) {  // none of this band's tiles is this part's
                        t += band_n;
                        continue;
                    }
                    for (int j = r.diag ? i0 * QD : 0; j < tb && next < g.count; ++j) {
                        const int ie = r.diag ? std::min(i1, j / QD + 1) : i1;  // rows with i * QD <= j
                        const int64_t cnt = ie - i0;  // the column's tiles: units [t, t + cnt)
                        for (; next < t + cnt; next += n_parts) emit(Unit{g.rect, i0 + (int)(next - t), j, g.cost});
                        t += cnt;
                    }
                }
            }
            at += g.count;
        }
    }
    while (si < side.size()) items.push_back(side[si++].w);  // the side items after the last main one
    auto work_cost = [&](const Work& w) { return (int64_t)(w.k1 - w.k0) * kChunk * kTile * TN; };
    // ---- the tail of the schedule: the last grid_cap items (the shortest, claimed last) are cut
    // into pieces along k so that the CTAs finish within a piece of each other.  Whole tiles of
    // ordinary rectangles (C2: makespan/mean 1.046 -> 1.005 in the planner's cost model) add their
    // pieces' partial counts into one slice per tile (red.global.add), which k2_tail_threshold
    // tests; k-pieces of accumulated rectangles are cut finer and add into their counters as before
    // (C3: 2,391 items of 22-24 chunks on 592 CTAs left 23 CTAs a fifth item, makespan/mean 1.22).
    const char* ate = getenv("BATMAP_K2_ACCTAIL");  // 0: no finer cut of accumulated tail pieces (test hook)
    const bool acc_tail_off = ate && ate[0] == '0';
    if (allow_split && grid_cap > 0 && !P.work.empty()) {
        WorkList& work = P.work;
        const size_t n = work.size();
        const size_t begin = n > (size_t)grid_cap ? n - (size_t)grid_cap : 0;
        std::vector<Work> pieces;
        int pcs = 0;
        for (size_t k = begin; k < n; ++k) {
            const Work w = work[k];
            const Rect& r = P.rects[w.rect];
            const int nk = r.W / kChunk;
            if (r.acc) {  // a k-piece of an accumulated rectangle: cut it finer, the counters add up
                const int len = w.k1 - w.k0;
                const int ap = acc_tail_off ? 1 : len >= 64 ? 8 : (len >= 16 ? 4 : (len >= 4 ? 2 : 1));
                for (int p = 0; p < ap; ++p) {
                    Work wp = w;
                    wp.k0 = w.k0 + (int32_t)((int64_t)len * p / ap);
                    wp.k1 = w.k0 + (int32_t)((int64_t)len * (p + 1) / ap);
                    if (p == 0) work[k] = wp;
                    else pieces.push_back(wp);
                }
                continue;
            }
            if (pcs == 0) pcs = nk >= 64 ? 8 : (nk >= 16 ? 4 : (nk >= 4 ? 2 : 1));
            if (pcs < 2 || w.k0 != 0 || w.k1 != nk || nk < 2 * pcs) continue;
            const int t = (int)P.tails.size();
            P.tails.push_back({w.rect, w.ti, w.tj, 0});
            for (int p = 0; p < pcs; ++p) {
                Work wp = w;
                wp.k0 = (int32_t)((int64_t)nk * p / pcs);
                wp.k1 = (int32_t)((int64_t)nk * (p + 1) / pcs);
                wp.tail = 1 + t * pcs + p;
                if (p == 0) work[k] = wp;
                else pieces.push_back(wp);
            }
        }
        if (!P.tails.empty()) P.tail_pieces = pcs;
        if (!pieces.empty()) {  // everything before `begin` costs at least as much: re-sort the tail only
            WorkList tail(work.begin() + (long)begin, work.end());
            tail.insert(tail.end(), pieces.begin(), pieces.end());
            stable_sort_desc(tail, work_cost);
            work.resize(begin);
            work.insert(work.end(), tail.begin(), tail.end());
        }
    }
    // ---- ordinary tiles that K2 will run in balanced mode (ragged or diagonal tiles whose warps hold
    // unequal numbers of valid blocks; k2_balance_pays, plan.h): they add their partial counts into a
    // tail slice like the cut tail tiles, and k2_tail_threshold tests them.  Scanned only for plans of
    // moderate size (C2: 5,312 items, 1.5 % of its K2 time in such tiles); in C4's 3e5 items they
    // weigh 0.2 % and the scan would lengthen the build.
    const char* be = getenv("BATMAP_K2_BALANCE");
    if (allow_split && !(be && be[0] == '0') && P.work.size() <= 65536) {
        const int pcs = P.tail_pieces > 0 ? P.tail_pieces : 1;
        for (Work& w : P.work) {
            if (w.tail) continue;
            const Rect& r = P.rects[w.rect];
            if (r.acc) continue;
            const bool ragged = (int64_t)(w.ti + 1) * kTile > r.n_rows || (int64_t)(w.tj + 1) * TN > r.n_cols ||
                                (r.diag && (int64_t)w.tj * TN < (int64_t)(w.ti + 1) * kTile);
            if (!ragged || !k2_balance_pays(r.n_rows, r.n_cols, r.diag, w.ti, w.tj, TN)) continue;
            const int t = (int)P.tails.size();
            P.tails.push_back({w.rect, w.ti, w.tj, 0});
            w.tail = 1 + t * pcs;
        }
        if (!P.tails.empty()) P.tail_pieces = pcs;
    }
}

}  // namespace bm

namespace bm {

// Tile width of a selection's plan: 64-column tiles when the cost model says they execute > 10 %
// fewer compares (small or ragged width classes) and there is enough work for the shape to matter
// (> 1e9 compares, ~0.1 ms); else 128.  Measured: C3 K2 1.28 -> 1.07 ms with 64; C1 (1.4e8
// compares, latency-bound) 0.061 -> 0.065 ms, hence the floor; C2 14.67 -> 14.90 ms (kept at 128 by
// the rule).  BATMAP_K2_TN=64|128 overrides.
int choose_tn(const std::vector<ClassInfo>& cls, bool allow_virtual, bool allow_promote) {
    const char* e = getenv("BATMAP_K2_TN");
    if (e && atoi(e) == 64) return 64;
    if (e && atoi(e) == 128) return kTile;
    const int64_t c128 = plan_cost(cls, allow_virtual, allow_promote, kTile);
    if (c128 < 1000000000ll) return kTile;
    const int64_t c64 = plan_cost(cls, allow_virtual, allow_promote, 64);
    return c64 * 10 < c128 * 9 ? 64 : kTile;
}

}  // namespace bm
