"""Pins for oracle/batmap_ref.py (the BatMap method step by step).

Independent anchors: the paper's worked width/throughput example, the
paper's Fig. 5 indicator assignments, the per-byte meaning of the count
condition checked exhaustively against the SWAR closed form, the
build invariants stated in §2 (two copies in two tables, exactly one counted), the
survey's independently derived golden bytes, and -- end to end --
the definition |S_i ∩ S_j| computed by sorted merge.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import batmap_ref as br
from workloads import uniform


def test_derive_params_and_width_paper_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "paper_throughput.json")))
    m = g["instance_size"] / (g["n_items"] * g["p"])  # 10^7 occurrences, 4000 items, 5%
    assert m == g["m_derived"] == 50_000
    s, U = br.derive_params(int(m))
    assert (s, U) == (9, 65024)  # 127·2^8 < 50,000 <= 127·2^9
    r = br.table_range(g["avg_set_size"], s, 128)
    assert r == g["r"] and 3 * r == g["batmap_width_bytes"]  # P:575 "3·2^13 bytes wide"
    # 4000^2 · 3·2^13 bytes in 10.87 s = 36.2 GB/s
    assert round(g["n_items"] ** 2 * 3 * r / g["seconds"] / 1e9, 1) == g["gbytes_per_s"]
    # 4000^2 · 2500 = 4·10^10 elements -> 3.68·10^9 elements/s
    assert g["n_items"] ** 2 * g["avg_set_size"] == g["elements_total"]
    assert round(g["elements_total"] / g["seconds"] / 1e9, 2) == g["elements_per_s"] / 1e9
    # merge microbenchmark rates
    assert round(2 * 2 ** 24 * 100 / g["merge_1core_seconds"] / 1e8, 2) == 2.25
    assert round(8 * 2 * 2 ** 24 * 100 / g["merge_8core_seconds"] / 1e9, 2) == 1.71


@pytest.mark.parametrize("m,s", [(1, 0), (127, 0), (128, 1), (254, 1), (255, 2), (10_000, 7),
                                 (100_000, 10), (1_000_000, 13), (200_000, 11)])
def test_derive_params_minimal(m, s):
    s2, U = br.derive_params(m)
    assert s2 == s and U >= m and (s == 0 or 127 * 2 ** (s - 1) < m)
    assert (U - 1) >> s == 126  # codes 0..126; 127 reserved for ⊥ (reading #1)


def test_table_range():
    assert br.table_range(1, 0, 64) == 64
    assert br.table_range(300, 9, 64) == 1024
    assert br.table_range(0, 7, 128) == 128
    for size in [1, 5, 63, 64, 65, 1000, 4096, 4097]:
        r = br.table_range(size, 0, 1)
        assert r & (r - 1) == 0 and r >= 2 * size and r < 4 * size + 1


@pytest.mark.parametrize("s", [0, 1, 3, 7, 10])
def test_pi_bijective_nonaffine(s):
    U = 127 * 2 ** s
    for seed in (0, 42):
        P = br.pi_table(seed, s)
        for t in range(3):
            assert np.array_equal(np.sort(P[t]), np.arange(U))  # permutation of [0, U)
        d = np.diff(P[0].astype(np.int64)) % U
        assert len(np.unique(d)) > 3  # not x -> a x + c mod U
    assert not np.array_equal(br.pi_table(0, s), br.pi_table(1, s))


def test_slot_formula_and_alignment():
    # direct evaluation of P:378-379 (SPEC S:141-142 examples)
    assert br.h(2, 677, 64, 64) == 101
    assert br.h(1, 677, 256, 64) == 421
    assert br.h(1, 0, 128, 128) == 0
    # for r_i | r_j, positions align: h^(j) mod 3r_i == h^(i)  (reading #18)
    rng = np.random.default_rng(0)
    for _ in range(2000):
        r0 = 2 ** int(rng.integers(2, 8))
        ri = r0 * 2 ** int(rng.integers(0, 4))
        rj = ri * 2 ** int(rng.integers(0, 4))
        v = int(rng.integers(0, 1 << 20))
        t = int(rng.integers(1, 4))
        assert br.h(t, v, rj, r0) % (3 * ri) == br.h(t, v, ri, r0)
        assert br.table_of(br.h(t, v, rj, r0), r0) == t


def test_indicator_fig5(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "paper_throughput.json")))["swar_fig5"]
    for a in g["assignments"]:
        t1, t2 = a["tables"]
        assert br.indicator(t1, t2) == a["bit"][str(t1)]
        assert br.indicator(t2, t1) == a["bit"][str(t2)]
        assert br.indicator(t1, t2) + br.indicator(t2, t1) == 1
    with pytest.raises(ValueError):
        br.indicator(2, 2)


def test_encode_entry():
    assert br.encode_entry(0, 0) == 0x00 and br.encode_entry(5, 1) == 0x85 and br.encode_entry(126, 0) == 0x7E
    with pytest.raises(ValueError):
        br.encode_entry(127, 0)


def _byte_rule(a, b):
    """Count condition of P:233 on one byte lane: equal element bits and b_i OR b_j."""
    return ((a & 0x7F) == (b & 0x7F)) & (((a | b) & 0x80) != 0)


def test_swar_exhaustive_per_lane():
    """P:426-430 vs the per-byte rule, all 65,536 byte pairs in each of the 4 lanes."""
    rng = np.random.default_rng(7)
    a = np.repeat(np.arange(256, dtype=np.uint64), 256)
    b = np.tile(np.arange(256, dtype=np.uint64), 256)
    for lane in range(4):
        ox = rng.integers(0, 2 ** 32, size=a.shape[0], dtype=np.uint64)
        oy = rng.integers(0, 2 ** 32, size=a.shape[0], dtype=np.uint64)
        sh = np.uint64(8 * lane)
        keep = ~(np.uint64(0xFF) << sh) & np.uint64(0xFFFFFFFF)
        x = (ox & keep) | (a << sh)
        y = (oy & keep) | (b << sh)
        got = br.swar_count_np(x, y)
        ref = np.zeros_like(got)
        for k in range(4):
            kk = np.uint64(8 * k)
            ref += _byte_rule((x >> kk) & np.uint64(0xFF), (y >> kk) & np.uint64(0xFF)).astype(np.int64)
        np.testing.assert_array_equal(got, ref)
    # SPEC S:243-245 examples
    assert br.swar_count(0x7F7F7F7F, 0x7F7F7F7F) == 0
    assert br.swar_count(0x7F7F7F85, 0x7F7F7F05) == 1
    assert br.swar_count(0x85858585, 0x05050505) == 4
    # 10^6 random words
    x = rng.integers(0, 2 ** 32, size=10 ** 6, dtype=np.uint64)
    y = np.where(rng.random(10 ** 6) < 0.5, x ^ rng.integers(0, 2, size=10 ** 6, dtype=np.uint64) * np.uint64(0x80),
                 rng.integers(0, 2 ** 32, size=10 ** 6, dtype=np.uint64))
    ref = sum(_byte_rule((x >> np.uint64(8 * k)) & np.uint64(0xFF), (y >> np.uint64(8 * k)) & np.uint64(0xFF)).astype(np.int64)
              for k in range(4))
    np.testing.assert_array_equal(br.swar_count_np(x, y), ref)


def _check_invariants(bm: br.BatMap):
    """§2 invariants."""
    ent = bm.encode()
    stored = set(bm.S) - set(bm.failed)
    assert len(bm.S) == bm.live + len(bm.failed)
    assert not (set(bm.failed) & stored)
    for x in stored:
        cps = bm.copies(x)
        assert len(cps) == 2  # stored in exactly two of the three tables
        bits = [ent[bm.pos(t, x)] >> 7 for t in cps]
        assert sum(bits) == 1  # one copy carries b = 1 (Fig. 5)
    for x in bm.failed:
        assert bm.copies(x) == []
    assert int((ent != br.NULL).sum()) == 2 * bm.live
    # decode: (slot, code) determines π_t(x) and that element is in S
    inv = [dict((int(v), x) for x, v in enumerate(bm.pi[t])) for t in range(3)]
    for q in np.flatnonzero(ent != br.NULL):
        t = br.table_of(int(q), bm.r0)
        # recover π_t(x): high bits from the code, low bits from the position
        g, o = divmod(int(q) % (3 * bm.r0 * (bm.r // bm.r0)), 3 * bm.r0)
        low = g * bm.r0 + (o - (t - 1) * bm.r0)  # = π mod r
        code = int(ent[q]) & 0x7F
        cands = [v for v in range(code << bm.s, (code + 1) << bm.s) if v % bm.r == low]
        assert len(cands) == 1  # unique reconstruction needs r >= 2^s
        assert inv[t - 1][cands[0]] in stored


@pytest.mark.parametrize("seed", range(6))
def test_build_invariants_random(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.choice([300, 5000, 60000]))
    s, _ = br.derive_params(m)
    P = br.pi_table(seed, s)
    pil = [P[t].tolist() for t in range(3)]
    size = int(rng.integers(1, min(m, 700)))
    S = np.sort(rng.choice(m, size=size, replace=False))
    r = br.table_range(size, s, 128)
    r0 = 128 if seed % 2 else r
    bm = br.BatMap(S, r, r0, pil, s).build()
    _check_invariants(bm)
    # count(B, B) = live
    w = br.words(bm.encode())
    assert br.count_pair(w, w) == bm.live


def test_forced_failures_invariants():
    m = 5000
    s, _ = br.derive_params(m)
    P = br.pi_table(3, s)
    pil = [P[t].tolist() for t in range(3)]
    S = np.arange(0, 4000, 7)
    bm = br.BatMap(S, br.table_range(len(S), s, 128), 128, pil, s, max_loop=1).build()
    assert len(bm.failed) > 0
    _check_invariants(bm)


def test_golden_c6(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "c6_batmap.json")))
    U = g["U"]
    pi = np.array([[(a * x + c) % U for x in range(U)] for a, c in g["pi_affine"]])
    names = ["A", "B", "C"]
    tids = np.concatenate([g["sets"][k] for k in names])
    off = np.zeros(4, np.int64)
    off[1:] = np.cumsum([len(g["sets"][k]) for k in names])
    col = br.Collection(off, tids, g["m"], r_min=g["r_min"], pi=pi)
    assert col.s == g["s"] and col.r0 == g["r0"]
    for i, k in enumerate(names):
        assert col.r[i] == g["r"][k]
        assert col.maps[i].failed == g["failed"][k]
        assert " ".join("%02X" % v for v in col.bytes[i]) == g["bytes"][k]
    assert ["0x%08X" % w for w in col.words[0]] == g["words_A"]
    for pair, val in g["raw_counts"].items():
        assert col.raw_count(names.index(pair[0]), names.index(pair[1])) == val
    sup = {(names[i], names[j]): int(s) for i, j, s in col.pair_supports(threshold=0)}
    for pair, val in g["supports"].items():
        assert sup[(pair[0], pair[1])] == val
    # and the supports are the definition
    np.testing.assert_array_equal(col.pair_supports(threshold=0), oracle.pairs_merge(off, tids, threshold=0))
    fo = g["failure_only"]
    ident = [list(range(U))] * 3
    bm = br.BatMap(fo["S"], fo["r"], fo["r0"], ident, 0, fo["max_loop"]).build()
    assert bm.failed == fo["failed"]
    assert " ".join("%02X" % v for v in bm.encode()) == fo["bytes"]


def _mixed_instance(seed):
    """Sets with sizes spanning ratios up to 64x (so r_i spans several classes)."""
    rng = np.random.default_rng(seed)
    m = int(rng.choice([2000, 20000, 65536]))
    n = int(rng.integers(6, 14))
    rows = []
    for i in range(n):
        size = int(min(m - 1, max(1, round(rng.uniform(4, 600) * 2 ** rng.integers(0, 5) / 4))))
        base = np.sort(rng.choice(m, size=size, replace=False))
        if i and rng.random() < 0.5:  # correlated sets so intersections are non-trivial
            base = np.unique(np.concatenate([base, rows[-1][: size // 2]]))
        rows.append(base.astype(np.int32))
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return off, np.concatenate(rows), m


@pytest.mark.parametrize("seed", range(8))
def test_end_to_end_equals_definition(seed):
    """count + corrections == |S_i ∩ S_j| on every pair."""
    off, tids, m = _mixed_instance(seed)
    max_loop = 1 if seed % 3 == 0 else None  # forced failures exercise M_{p,q}
    col = br.Collection(off, tids, m, seed=seed, r_min=128 if seed % 2 else 64, max_loop=max_loop)
    if max_loop == 1:
        assert col.failures()
    ref = oracle.pairs_merge(off, tids, threshold=0)
    np.testing.assert_array_equal(col.pair_supports(threshold=0), ref)
    # raw count alone is |stored_i ∩ stored_j|
    st = [set(S.tolist()) - set(bm.failed) for S, bm in zip(col.sets, col.maps)]
    for i in range(col.n):
        for j in range(i + 1, col.n):
            assert col.raw_count(i, j) == len(st[i] & st[j])


def test_end_to_end_colliding_pi():
    """An affine π forces systematic failures; corrections keep it exact."""
    off, tids = uniform(10, 3000, 0.1, 5)
    s, U = br.derive_params(3000)
    pi = np.array([[(a * x + c) % U for x in range(U)] for a, c in [(1, 0), (5, 3), (11, 7)]])
    col = br.Collection(off, tids, 3000, r_min=128, pi=pi)
    assert len(col.failures()) > 0
    np.testing.assert_array_equal(col.pair_supports(threshold=0), oracle.pairs_merge(off, tids, threshold=0))


def test_insertion_statistics():
    """§2.2: failures are rare and moves per insertion are O(1) (fewer trials)."""
    s, _ = br.derive_params(1 << 20)
    P = br.pi_table(11, s)
    pil = [P[t].tolist() for t in range(3)]
    rng = np.random.default_rng(11)
    fails, builds_ok, moves, ins = 0, 0, 0, 0
    for _ in range(4):
        S = np.sort(rng.choice(1 << 20, size=5000, replace=False))
        r = br.table_range(len(S), s, 128)
        bm = br.BatMap(S, r, r, pil, s).build()
        fails += len(bm.failed)
        builds_ok += not bm.failed
        moves += bm.moves
        ins += 2 * len(S)
    assert fails <= 0.01 * ins
    assert moves / ins <= 10
    assert builds_ok >= 2


def test_memory_linearity():
    """Collection bytes = sum 3 r_i, with 3 r_i / |S_i| <= 12 when the size floor is inactive."""
    off, tids = uniform(30, 40000, 0.02, 9)
    col = br.Collection(off, tids, 40000, r_min=128)
    assert sum(len(b) for b in col.bytes) == sum(3 * r for r in col.r)
    for S, r in zip(col.sets, col.r):
        if len(S) >= max(2 ** col.s, 128) / 2:
            assert 3 * r / len(S) <= 12
    assert math.isclose(len(col.bytes[0]) / 3, col.r[0])
