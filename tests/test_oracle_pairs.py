"""Pins for the definition oracle (oracle/pairs.c): supp(i,j) = |S_i ∩ S_j|.

Each pin is independent of the oracle's own code: brute force straight from the
definition of support over transactions, the Gram matrix X^T X of the 0/1
incidence matrix (BLAS dgemm, exact below 2^53), the invariant
sum_{i<j} supp(i,j) = sum_b C(|T_b|, 2), and SPEC's worked examples.
"""
import itertools

import numpy as np
import pytest

import oracle
from workloads import make_config, to_horizontal, uniform


def _random_tiny(rng, n, m, p):
    rows = [np.flatnonzero(rng.random(m) < p).astype(np.int32) for _ in range(n)]
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows) if rows else np.empty(0, np.int32)
    return off, tids.astype(np.int32)


def _brute(off, tids, m, threshold, items=None):
    """Count, for every pair {i,j}, the transactions T_b that contain both."""
    n = off.shape[0] - 1
    sel = sorted(set(range(n) if items is None else items))
    T = [set() for _ in range(m)]
    for i in range(n):
        for b in tids[off[i]:off[i + 1]]:
            T[int(b)].add(i)
    out = []
    for i, j in itertools.combinations(sel, 2):
        s = sum(1 for b in range(m) if i in T[b] and j in T[b])
        if s >= threshold:
            out.append((i, j, s))
    return np.array(out, dtype=np.uint32).reshape(-1, 3)


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_tiny(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 13))
    m = int(rng.integers(1, 65))
    p = float(rng.uniform(0.05, 0.8))
    off, tids = _random_tiny(rng, n, m, p)
    for thr in (0, 1, 2, 3):
        ref = _brute(off, tids, m, thr)
        np.testing.assert_array_equal(oracle.pairs_merge(off, tids, threshold=thr), ref)
        np.testing.assert_array_equal(oracle.pairs_horizontal(off, tids, m, threshold=thr), ref)
    items = sorted(rng.choice(n, size=max(1, n // 2), replace=False).tolist())
    ref = _brute(off, tids, m, 1, items)
    np.testing.assert_array_equal(oracle.pairs_merge(off, tids, items=items, threshold=1), ref)
    np.testing.assert_array_equal(oracle.pairs_horizontal(off, tids, m, items=items, threshold=1), ref)


def _gram(off, tids, m):
    n = off.shape[0] - 1
    X = np.zeros((m, n), dtype=np.float64)
    X[tids, np.repeat(np.arange(n), np.diff(off))] = 1.0
    return np.rint(X.T @ X).astype(np.int64)


@pytest.mark.parametrize("n,m,p,seed", [(40, 500, 0.2, 1), (300, 3000, 0.02, 2), (120, 2000, 0.5, 3)])
def test_gram_matrix(n, m, p, seed):
    off, tids = uniform(n, m, p, seed)
    G = _gram(off, tids, m)
    iu, ju = np.triu_indices(n, 1)
    for res in (oracle.pairs_merge(off, tids, threshold=0), oracle.pairs_horizontal(off, tids, m, threshold=0)):
        assert res.shape[0] == n * (n - 1) // 2
        np.testing.assert_array_equal(res[:, 0], iu)
        np.testing.assert_array_equal(res[:, 1], ju)
        np.testing.assert_array_equal(res[:, 2].astype(np.int64), G[iu, ju])
    # diagonal of the Gram matrix is |S_i|
    np.testing.assert_array_equal(np.diag(G), np.diff(off))


def test_gram_c1_thresholded():
    w = make_config("C1")
    G = _gram(w.offsets, w.tids, w.m)
    iu, ju = np.triu_indices(w.n, 1)
    keep = G[iu, ju] >= w.threshold
    ref = np.stack([iu[keep], ju[keep], G[iu, ju][keep]], axis=1).astype(np.uint32)
    np.testing.assert_array_equal(oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=w.threshold), ref)
    np.testing.assert_array_equal(oracle.pairs_merge(w.offsets, w.tids, threshold=w.threshold), ref)
    assert 1000 < ref.shape[0] < 3000  # expected K ≈ 1.8e3 for C1


@pytest.mark.parametrize("cfg", ["C1"])
def test_sum_invariant(cfg):
    """sum_{i<j} supp(i,j) = sum_b C(|T_b|, 2) (north_star invariant)."""
    w = make_config(cfg)
    toff, _ = to_horizontal(w.offsets, w.tids, w.m)
    tl = np.diff(toff)
    expect = int((tl * (tl - 1) // 2).sum())
    res = oracle.pairs_horizontal(w.offsets, w.tids, w.m, threshold=1)
    assert int(res[:, 2].astype(np.int64).sum()) == expect


def test_spec_examples():
    # db = [{0,1},{0,1},{1}], threshold 2 -> {(0,1): 2}; threshold > m -> empty
    off = np.array([0, 2, 5], np.int64)
    tids = np.array([0, 1, 0, 1, 2], np.int32)
    for f in (lambda t: oracle.pairs_merge(off, tids, threshold=t),
              lambda t: oracle.pairs_horizontal(off, tids, 3, threshold=t)):
        np.testing.assert_array_equal(f(2), [[0, 1, 2]])
        assert f(4).shape == (0, 3)
    assert oracle.merge_count(np.array([1, 3, 5]), np.array([3, 5, 7])) == 2
    assert oracle.merge_count(np.array([1, 3, 5]), np.array([], np.int32)) == 0


def test_special_cases():
    # identical tidlists -> |S|; disjoint -> 0; supp <= min(|S_i|, |S_j|); symmetric
    a = np.arange(0, 100, 3, dtype=np.int32)
    b = np.arange(1, 100, 3, dtype=np.int32)
    off = np.array([0, len(a), 2 * len(a), 2 * len(a) + len(b)], np.int64)
    tids = np.concatenate([a, a, b])
    res = oracle.pairs_merge(off, tids, threshold=0)
    np.testing.assert_array_equal(res, [[0, 1, len(a)], [0, 2, 0], [1, 2, 0]])
    w = make_config("C1")
    res = oracle.pairs_merge(w.offsets, w.tids, threshold=1)
    sz = np.diff(w.offsets)
    assert (res[:, 2] <= np.minimum(sz[res[:, 0]], sz[res[:, 1]])).all()
    sym = oracle.merge_list(w.offsets, w.tids, res[:200, 1], res[:200, 0])
    np.testing.assert_array_equal(sym, res[:200, 2])


def test_merge_rows_sample_matches_full():
    w = make_config("C1")
    full = oracle.pairs_merge(w.offsets, w.tids, threshold=w.threshold)
    part = oracle.pairs_merge(w.offsets, w.tids, threshold=w.threshold, rows=(100, 200))
    np.testing.assert_array_equal(part, full[(full[:, 0] >= 100) & (full[:, 0] < 200)])


def test_empty_and_degenerate():
    off = np.array([0, 0, 0], np.int64)
    tids = np.empty(0, np.int32)
    np.testing.assert_array_equal(oracle.pairs_merge(off, tids, threshold=0), [[0, 1, 0]])
    assert oracle.pairs_horizontal(off, tids, 5, threshold=1).shape == (0, 3)
    one = np.array([0, 3], np.int64)
    assert oracle.pairs_merge(one, np.array([0, 1, 2], np.int32), threshold=0).shape == (0, 3)
