"""Pins for the NEXT-4 reference (oracle/batmap3_ref.py): 3-of-4 BatMaps for triples.

Independent of the module's own code: the exactly-once property of the counting rule (reading
#30) checked exhaustively over every combination of missing tables; the layout invariants of a
built BatMap (three copies per stored element at its designated slots, nothing else stored);
and end to end, raw count + corrections = |S_i ∩ S_j ∩ S_k| from the triple definition oracle
(three-finger merge, oracle/triples.c) on mixed-width instances -- with forced failures
(max_loop = 1) and with a colliding affine π.
"""
import itertools

import numpy as np
import pytest

import oracle
from oracle import batmap3_ref as b3


def test_params_and_layout_shape():
    assert b3.derive_params3(63) == (0, 63)
    assert b3.derive_params3(64) == (1, 126)
    assert b3.derive_params3(50_000) == (10, 63 * 1024)  # 63·2^9 = 32,256 < 50,000
    assert b3.table_range3(2500, 10, 128) == 8192
    r, r0 = 64, 16
    slots = {b3.h4(t, v, r, r0) for t in (1, 2, 3, 4) for v in range(r)}
    assert slots == set(range(4 * r))  # the four tables tile the 4r entries
    for t in (1, 2, 3, 4):
        for v in range(r):
            assert b3.table_of4(b3.h4(t, v, r, r0), r0) == t


def test_pi_tables_are_permutations():
    P = b3.pi_table4(7, 3)
    U = 63 * 8
    for t in range(4):
        assert sorted(P[t].tolist()) == list(range(U))
    assert not np.array_equal(P[0], P[1])


def test_counting_rule_counts_every_common_element_exactly_once():
    """For every (m_i, m_j, m_k) (the table each BatMap leaves out): summing reading #30's rule over
    the tables that hold x in all three gives exactly 1 -- with codes equal, any code."""
    for mi, mj, mk in itertools.product(range(1, 5), repeat=3):
        for code in (0, 17, 62):
            n = 0
            for t in (1, 2, 3, 4):
                if t in (mi, mj, mk):
                    continue
                a, b, c = (b3.encode_entry3(code, t, m) for m in (mi, mj, mk))
                n += b3.entry_counts(a, b, c, t)
            assert n == 1, (mi, mj, mk, code)


def test_counting_rule_never_counts_mismatch_or_null():
    rng = np.random.default_rng(0)
    for _ in range(20000):
        t = int(rng.integers(1, 5))
        ms = [int(rng.choice([u for u in (1, 2, 3, 4) if u != t])) for _ in range(3)]
        codes = [int(x) for x in rng.integers(0, 63, size=3)]
        if len(set(codes)) == 1:
            codes[2] = (codes[2] + 1) % 63
        e = [b3.encode_entry3(cd, t, m) for cd, m in zip(codes, ms)]
        assert not b3.entry_counts(*e, t)
    for t in (1, 2, 3, 4):
        assert not b3.entry_counts(b3.NULL3, b3.NULL3, b3.NULL3, t)


def _instance(seed, n=9, m=3000, max_size=700):
    rng = np.random.default_rng(seed)
    rows = []
    pool = rng.choice(m, size=max_size, replace=False)
    for _ in range(n):
        size = int(rng.integers(1, max_size))
        rows.append(np.unique(np.concatenate([rng.choice(pool, size=size // 2, replace=False),
                                              rng.choice(m, size=size - size // 2)])).astype(np.int32))
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return off, np.concatenate(rows), m


def _check_layout(c):
    for i, bm in enumerate(c.maps):
        f = set(bm.failed)
        stored = 0
        for x in bm.S:
            k = len(bm.copies(x))
            assert k == (0 if x in f else 3), (i, x, k)
            stored += k
        assert sum(v is not None for v in bm.A) == stored
        assert len(bm.S) == len(set(bm.S))


@pytest.mark.parametrize("seed,max_loop", [(0, None), (1, None), (2, 1), (3, 1), (4, 2)])
def test_count_plus_correction_is_the_triple_support(seed, max_loop):
    off, tids, m = _instance(seed)
    c = b3.Collection3(off, tids, m, seed=seed, r_min=64, max_loop=max_loop)
    _check_layout(c)
    if max_loop == 1:
        assert c.failures()
    tri = list(itertools.combinations(range(c.n), 3))
    got = c.triple_supports(tri)
    ti, tj, tk = (np.array(x, np.int32) for x in zip(*tri))
    np.testing.assert_array_equal(got, oracle.triples_list(off, tids, ti, tj, tk))


def test_colliding_affine_pi_forces_failures_and_stays_exact():
    off, tids, m = _instance(5, n=6, m=500, max_size=150)
    s3, U = b3.derive_params3(m)
    x = np.arange(U)
    pi = np.stack([(a * x + cc) % U for a, cc in ((1, 0), (5, 3), (11, 7), (13, 1))]).astype(np.int64)
    c = b3.Collection3(off, tids, m, r_min=4, pi=pi)
    assert c.failures()
    _check_layout(c)
    tri = list(itertools.combinations(range(c.n), 3))
    ti, tj, tk = (np.array(v, np.int32) for v in zip(*tri))
    np.testing.assert_array_equal(c.triple_supports(tri), oracle.triples_list(off, tids, ti, tj, tk))
