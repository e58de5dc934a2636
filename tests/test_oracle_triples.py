"""Pins for the NEXT-4 triple oracle (oracle/triples.c): supp(i,j,k) = |S_i ∩ S_j ∩ S_k| (P:43-44 for
itemsets of size 3; the paper leaves larger itemsets open).

Each pin is independent of the oracle's own code: brute force straight from the definition of
support over transactions; the third-order incidence contraction
supp(i,j,k) = sum_b X[b,i] X[b,j] X[b,k] (numpy einsum); the invariant
sum_{i<j<k} supp(i,j,k) = sum_b C(|T_b|, 3); monotonicity against the PAIR oracle
(supp(i,j,k) <= supp of each of its three pairs, the Apriori property the candidate generation
relies on); and special cases (identical sets, disjoint sets).
"""
import itertools
import math

import numpy as np
import pytest

import oracle
from workloads import to_horizontal, uniform


def _random_tiny(rng, n, m, p):
    rows = [np.flatnonzero(rng.random(m) < p).astype(np.int32) for _ in range(n)]
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows) if rows else np.empty(0, np.int32)
    return off, tids.astype(np.int32)


def _brute(off, tids, m, threshold, items=None):
    """Count, for every triple {i,j,k}, the transactions T_b that contain all three."""
    n = off.shape[0] - 1
    sel = sorted(set(range(n) if items is None else items))
    T = [set() for _ in range(m)]
    for i in range(n):
        for b in tids[off[i]:off[i + 1]]:
            T[int(b)].add(i)
    out = []
    for i, j, k in itertools.combinations(sel, 3):
        s = sum(1 for b in range(m) if i in T[b] and j in T[b] and k in T[b])
        if s >= max(threshold, 1):
            out.append((i, j, k, s))
    return np.array(out, dtype=np.uint32).reshape(-1, 4)


def test_three_finger_merge_examples():
    assert oracle.triple_count([1, 2, 3, 5], [2, 3, 5, 7], [0, 3, 5]) == 2
    assert oracle.triple_count([], [1], [1]) == 0
    assert oracle.triple_count([4], [4], [4]) == 1
    assert oracle.triple_count([1, 3, 5, 7, 9], [2, 4, 6, 8], [1, 2, 3]) == 0


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_tiny(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 11))
    m = int(rng.integers(1, 50))
    p = float(rng.uniform(0.1, 0.9))
    off, tids = _random_tiny(rng, n, m, p)
    for thr in (1, 2, 3):
        ref = _brute(off, tids, m, thr)
        np.testing.assert_array_equal(oracle.triples_horizontal(off, tids, m, threshold=thr), ref)
        if ref.shape[0]:
            np.testing.assert_array_equal(oracle.triples_list(off, tids, ref[:, 0], ref[:, 1], ref[:, 2]), ref[:, 3])
    items = sorted(rng.choice(n, size=max(3, n - 2), replace=False).tolist())
    np.testing.assert_array_equal(oracle.triples_horizontal(off, tids, m, items=items, threshold=1),
                                  _brute(off, tids, m, 1, items))


@pytest.mark.parametrize("seed", range(3))
def test_incidence_contraction(seed):
    off, tids = uniform(60, 400, 0.15, seed)
    m = 400
    X = np.zeros((m, 60), dtype=np.int64)
    for i in range(60):
        X[tids[off[i]:off[i + 1]], i] = 1
    G = np.einsum("bi,bj,bk->ijk", X, X, X)
    got = oracle.triples_horizontal(off, tids, m, threshold=1)
    assert np.array_equal(G[got[:, 0], got[:, 1], got[:, 2]], got[:, 3].astype(np.int64))
    # every triple i<j<k with G > 0 is emitted, nothing else
    iu = [(i, j, k) for i, j, k in itertools.combinations(range(60), 3) if G[i, j, k] > 0]
    assert len(iu) == got.shape[0]


def test_sum_invariant_and_pair_monotonicity():
    off, tids = uniform(120, 3000, 0.05, 11)
    m = 3000
    got = oracle.triples_horizontal(off, tids, m, threshold=1)
    toff, _ = to_horizontal(off, tids, m)
    sizes = np.diff(toff)
    assert int(got[:, 3].astype(np.int64).sum()) == sum(math.comb(int(s), 3) for s in sizes)
    pairs = oracle.pairs_merge(off, tids, threshold=0)
    P = {(int(a), int(b)): int(s) for a, b, s in pairs}
    for i, j, k, s in got[:: max(1, got.shape[0] // 2000)]:
        assert s <= min(P[(i, j)], P[(i, k)], P[(j, k)])
    np.testing.assert_array_equal(oracle.triples_list(off, tids, got[:, 0], got[:, 1], got[:, 2]), got[:, 3])


def test_special_cases():
    S = np.arange(0, 500, 3, dtype=np.int32)
    off = np.array([0, len(S), 2 * len(S), 3 * len(S), 3 * len(S) + 2], np.int64)
    tids = np.concatenate([S, S, S, np.array([1, 2], np.int32)])
    got = oracle.triples_horizontal(off, tids, 500, threshold=1)
    np.testing.assert_array_equal(got, np.array([[0, 1, 2, len(S)]], np.uint32))  # identical sets -> |S|
    assert oracle.triple_count(S, S + 1, S) == 0  # disjoint -> 0
    with pytest.raises(ValueError):
        oracle.triples_horizontal(np.zeros(5000, np.int64), np.zeros(0, np.int32), 10)
