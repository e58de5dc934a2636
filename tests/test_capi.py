"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol
include/batmap.h declares, rejects bad arguments without touching the device, and its
host-only planner partitions the pair triangle exactly."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    hdr = open(os.path.join(ROOT, "include", "batmap.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:batmap_status|void|const char\*)\s+(batmap_\w+)\s*\(", hdr, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1102_1003_b200 import batmap

    lib = batmap.load_library()
    names = _declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    raw = ctypes.CDLL(batmap.LIB_PATH)
    for n in names:
        getattr(raw, n)
    assert batmap.version().startswith("batmap-b200")


def test_library_is_sm100a_only():
    from paper_1102_1003_b200 import batmap
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", batmap.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    dump = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", batmap.LIB_PATH],
                          capture_output=True, text=True).stdout
    funcs = dump.split("Function : ")
    k2 = [f for f in funcs if f.startswith("_ZN2bm8k2_tiled")]
    assert k2, "tiled intersection kernel missing"
    sass = "".join(k2)
    assert "UTMALDG" in sass  # TMA (cp.async.bulk.tensor) in the intersection kernel
    assert "IDP.4A" in sass and "LOP3" in sass


def test_argument_errors_without_device():
    from paper_1102_1003_b200 import batmap

    lib = batmap.load_library()
    h = ctypes.c_void_p()
    assert lib.batmap_build(None, None, 3, 10, None, None, ctypes.byref(h)) == batmap.BATMAP_E_INVALID
    assert b"NULL" in lib.batmap_last_error()
    assert lib.batmap_build(ctypes.c_void_p(8), ctypes.c_void_p(8), 3, 1 << 31, None, None,
                            ctypes.byref(h)) == batmap.BATMAP_E_OVERFLOW
    o = batmap.BuildOpts()
    o.r_min = 96
    assert lib.batmap_build(ctypes.c_void_p(8), ctypes.c_void_p(8), 3, 10, ctypes.byref(o), None,
                            ctypes.byref(h)) == batmap.BATMAP_E_INVALID
    n = ctypes.c_int64()
    assert lib.batmap_pair_supports(None, None, 0, 1, None, 0, ctypes.byref(n), None) == batmap.BATMAP_E_INVALID
    inf = batmap.Info()
    assert lib.batmap_info(None, ctypes.byref(inf)) == batmap.BATMAP_E_INVALID
    lib.batmap_destroy(None)
    fh, bad = ctypes.c_void_p(), ctypes.c_int64()
    assert lib.batmap_fimi_parse(None, 5, None, ctypes.byref(fh), ctypes.byref(bad)) == batmap.BATMAP_E_INVALID
    assert lib.batmap_fimi_parse(ctypes.c_void_p(8), -1, None, ctypes.byref(fh), ctypes.byref(bad)) == \
        batmap.BATMAP_E_INVALID
    assert lib.batmap_fimi_filter(None, 3, None) == batmap.BATMAP_E_INVALID
    assert lib.batmap_fimi_info(None, ctypes.byref(n), ctypes.byref(n), ctypes.byref(n)) == batmap.BATMAP_E_INVALID
    assert lib.batmap_frequent_items(None, 5, 1, None, ctypes.byref(n), None) == batmap.BATMAP_E_INVALID
    assert lib.batmap_frequent_items(ctypes.c_void_p(8), -1, 1, ctypes.c_void_p(8), ctypes.byref(n), None) == \
        batmap.BATMAP_E_INVALID
    lib.batmap_fimi_destroy(None)


def _collect(class_n, class_w, n_parts, grid_cap=0):
    from paper_1102_1003_b200 import plan_work

    parts = [plan_work(class_n, class_w, p, n_parts, grid_cap) for p in range(n_parts)]
    return parts


def _planned(class_n, class_w):
    """Planned classes (promotion merges runs of adjacent classes): (n, W, group_of)."""
    from paper_1102_1003_b200 import plan_groups

    g = plan_groups(class_n, class_w).tolist()
    assert g == sorted(g) and g[0] == 0 and all(b - a in (0, 1) for a, b in zip(g, g[1:]))
    pn = [sum(n for n, gg in zip(class_n, g) if gg == e) for e in range(g[-1] + 1)]
    pw = [max(w for w, gg in zip(class_w, g) if gg == e) for e in range(g[-1] + 1)]
    return pn, pw, g


@pytest.mark.parametrize("class_n,class_w", [([1000], [96]), ([780, 220], [192, 384]),
                                             ([2000, 40, 30, 20, 10, 5, 3, 1], [96 * 2 ** k for k in range(8)]),
                                             ([300, 200, 120, 90, 50, 12], [96 * 2 ** k for k in range(6)]),
                                             ([1, 7, 100, 454, 427, 11], [768 * 2 ** k for k in range(6)]),
                                             ([5], [96])])
@pytest.mark.parametrize("n_parts", [1, 2, 3, 8])
def test_plan_work_partition_exact(class_n, class_w, n_parts):
    """Union over parts = every k-chunk of every tile of the (planned-class) pair triangle exactly
    once; tile rows of accumulated rectangles stay on one part; algorithmic work adds
    up to sum_{i<j} max(W_i, W_j) over the ORIGINAL widths."""
    from paper_1102_1003_b200 import plan_tile

    parts = _collect(class_n, class_w, n_parts)
    pn, pw, _ = _planned(class_n, class_w)
    tr, tc = plan_tile(class_n, class_w)
    assert tr == 128 and tc in (64, 128)
    chunks = {}
    rect_R = {}
    row_part = {}
    for p, (items, wc, tcmp) in enumerate(parts):
        assert tcmp == int(sum((k1 - k0) * 16 * 128 * tc for _, _, _, _, k0, k1, _, _ in items.tolist()))
        for a, b, ti, tj, k0, k1, R, acc in items.tolist():
            assert a <= b and k0 < k1
            rect_R.setdefault((a, b), (R, acc))
            assert rect_R[(a, b)] == (R, acc)
            for k in range(k0, k1):
                key = (a, b, ti, tj, k)
                assert key not in chunks
                chunks[key] = p
            if acc:
                assert row_part.setdefault((a, b, ti), p) == p
    expect = set()
    C = len(pn)
    for a in range(C):
        for b in range(a, C):
            if pn[a] == 0 or pn[b] == 0 or (a == b and pn[a] < 2):
                continue
            R, _ = rect_R[(a, b)]
            W = pw[b] // R
            ta = -(-pn[a] // 128)
            tb = -(-(pn[b] * R) // tc)
            for i in range(ta):
                for j in range(i * 128 // tc if a == b else 0, tb):
                    for k in range(W // 16):
                        expect.add((a, b, i, j, k))
    assert set(chunks) == expect
    wc_total = sum(wc for _, wc, _ in parts)
    C = len(class_n)
    closed = sum(class_n[a] * class_n[b] * class_w[b] for a in range(C) for b in range(a + 1, C))
    closed += sum(n * (n - 1) // 2 * w for n, w in zip(class_n, class_w))
    assert wc_total == closed


def test_plan_groups_promotion(monkeypatch):
    """Small narrow classes are merged into a planned class of their widest member's width (the
    T40I10D100K-shaped C3 classes: 1, 7 and 100 items of 768 ... 3072 words); large classes stay
    apart; BATMAP_K2_PROMOTE=0 disables it; executed work drops."""
    from paper_1102_1003_b200 import plan_groups

    cn, cw = [1, 7, 100, 454, 427, 11], [768 * 2 ** k for k in range(6)]
    g = plan_groups(cn, cw).tolist()
    assert g[0] == g[1] == g[2] and len(set(g)) >= 3
    assert plan_groups([7822, 2178], [1536, 3072]).tolist() == [0, 1]  # C2: nothing to gain
    _, wc1, tc1 = _collect(cn, cw, 1)[0]
    monkeypatch.setenv("BATMAP_K2_PROMOTE", "0")
    assert plan_groups(cn, cw).tolist() == list(range(6))
    _, wc0, tc0 = _collect(cn, cw, 1)[0]
    assert wc0 == wc1 and tc1 < 0.85 * tc0


def test_plan_work_virtual_and_split():
    """Skinny rectangles are virtualised (R = W_b / W_a) and long tiles split along k."""
    parts = _collect([99835, 1], [6144, 6144 * 256], 1)
    items = parts[0][0]
    skinny = items[(items[:, 0] == 0) & (items[:, 1] == 1)]
    assert (skinny[:, 6] == 256).all() and (skinny[:, 7] == 1).all()
    items = _collect([50, 40], [24576, 49152], 1)[0][0]  # few long tiles -> split-K
    assert (items[:, 7] == 1).any() and (items[:, 5] - items[:, 4] < 49152 // 16).any()


@pytest.mark.parametrize("tn", ["", "64", "128"])
def test_plan_work_covers_every_pair_once(tn, monkeypatch):
    """Expanding the work items (virtual columns, k-chunks, promoted classes) covers, for every pair
    i < j, each of the K words of its planned column item exactly once, with K a power-of-two
    multiple of max(W_i, W_j): c_ij = sum_{w < W_j} SWAR(B_j[w], B_i[w mod W_i]),
    counted K / max(W_i, W_j) times and divided exactly."""
    from paper_1102_1003_b200 import plan_tile

    if tn:
        monkeypatch.setenv("BATMAP_K2_TN", tn)
    for class_n, class_w in (([130, 7, 3], [16, 64, 256]), ([3, 5, 140, 2], [16, 32, 64, 128]),
                             ([200, 90], [32, 64])):
        pn, pw, g = _planned(class_n, class_w)
        tc = plan_tile(class_n, class_w)[1]
        first = np.cumsum([0] + pn)
        items = _collect(class_n, class_w, 1)[0][0]
        cover = {}
        for a, b, ti, tj, k0, k1, R, acc in items.tolist():
            Wv = pw[b] // R
            for r in range(ti * 128, min(pn[a], ti * 128 + 128)):
                for v in range(tj * tc, min(pn[b] * R, tj * tc + tc)):
                    j, rep = divmod(v, R)
                    if a == b and r >= j:
                        continue
                    key = (first[a] + r, first[b] + j)
                    for k in range(k0 * 16, k1 * 16):
                        w = rep * Wv + k  # word of (planned) B_j
                        cover[(key, w)] = cover.get((key, w), 0) + 1
        n = sum(class_n)
        pairs = {(i, j) for i in range(n) for j in range(i + 1, n)}
        assert {k for k, _ in cover} == pairs
        assert set(cover.values()) == {1}
        width, pwidth = {}, {}
        pos = 0
        for a in range(len(class_n)):
            for r in range(class_n[a]):
                width[pos] = class_w[a]
                pwidth[pos] = pw[g[a]]
                pos += 1
        per_pair = {}
        for (key, w) in cover:
            per_pair[key] = per_pair.get(key, 0) + 1
        for (i, j), cnt in per_pair.items():
            K = pwidth[j]
            assert cnt == K and K % max(width[i], width[j]) == 0
            q = K // max(width[i], width[j])
            assert q & (q - 1) == 0


def test_cli_builds_and_prints_usage():
    """The native command-line miner (cli/batmap_mine.cpp, C ABI only) is built next to the library
    and links it; without arguments it prints its usage and exits 2 (no device touched)."""
    import subprocess

    from paper_1102_1003_b200 import build_ext

    exe = build_ext.build_cli()
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr
    r = subprocess.run([exe, "/nonexistent.dat", "0"], capture_output=True, text=True)
    assert r.returncode == 2  # min_support 0 rejected before any I/O


def test_plan_work_grouped_tile_order(monkeypatch):
    """Tiles of an ordinary rectangle come in bands of G tile rows (column by column inside a band),
    G = 32 MB / (128 W_a 4 B): the first grid of CTAs shares a band of row tiles, and each column
    tile streams from HBM once per band.  BATMAP_K2_GROUP=1 is row-major.  Same tiles either way."""
    cn, cw = [6000], [6144]  # C4's narrow class shape: 3 MB per tile row -> G = 10
    items = _collect(cn, cw, 1)[0][0]
    first = items[:296]
    assert set(first[:, 2].tolist()) == set(range(10))  # ti in the first band
    assert (np.diff(first[:, 3]) >= 0).all()  # columns ascend inside the band
    monkeypatch.setenv("BATMAP_K2_GROUP", "1")
    rows = _collect(cn, cw, 1)[0][0]
    assert (rows[:40, 2] == 0).all() and (rows[:40, 3] == np.arange(40)).all()
    # the same tiles (the last grid's worth may be cut into k-pieces differently)
    assert np.array_equal(np.unique(items[:, :4], axis=0), np.unique(rows[:, :4], axis=0))
