"""NEXT-4 on the GPU, through the C-ABI: 3-of-4 BatMaps and triple supports (readings
#26-#32) against the oracles.

* the serial build writes exactly the reference's bytes (oracle/batmap3_ref.py), also with a
  colliding affine π and forced failures;
* every concurrent build satisfies the layout invariants (three copies per stored element at
  its designated slots, the entry bits of reading #29, nothing else stored);
* triple supports equal the definition (oracle/triples.c) on every candidate, with failures;
* the Apriori candidates equal the brute-force join of the pair list;
* frequent triples end to end (mine_triples) equal horizontal triple counting on C1, C3 and a
  planted instance.
"""
import itertools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import batmap3_ref as b3  # noqa: E402
from workloads import make_config, uniform  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1102_1003_b200 import batmap

    batmap.load_library()


def _c3(off, tids, m, **kw):
    from paper_1102_1003_b200 import Collection3

    return Collection3(torch.as_tensor(off, dtype=torch.int64).cuda(), torch.as_tensor(tids, dtype=torch.int32).cuda(),
                       m, **kw)


def _instance(seed, n=10, m=3000, max_size=700):
    rng = np.random.default_rng(seed)
    pool = rng.choice(m, size=max_size, replace=False)
    rows = []
    for _ in range(n):
        size = int(rng.integers(1, max_size))
        rows.append(np.unique(np.concatenate([rng.choice(pool, size=size // 2, replace=False),
                                              rng.choice(m, size=size - size // 2)])).astype(np.int32))
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return off, np.concatenate(rows), m


def _all_triples(n):
    return np.array(list(itertools.combinations(range(n), 3)), dtype=np.int32).reshape(-1, 3)


@pytest.mark.parametrize("seed,max_loop", [(0, 0), (1, 0), (2, 1), (3, 2)])
def test_serial_build_bytes_equal_reference(seed, max_loop):
    off, tids, m = _instance(seed)
    ref = b3.Collection3(off, tids, m, seed=seed, r_min=128, max_loop=max_loop or None)
    c = _c3(off, tids, m, seed=seed, max_loop=max_loop, serial=True)
    for i in range(len(off) - 1):
        np.testing.assert_array_equal(c.export_entries(i), ref.bytes[i])
    got_f = c.failures()
    assert [tuple(x) for x in got_f.tolist()] == ref.failures()
    if max_loop == 1:
        assert len(ref.failures()) > 0


def test_colliding_affine_pi_bytes_and_supports():
    off, tids, m = _instance(5, n=7, m=500, max_size=150)
    s3, U = b3.derive_params3(m)
    x = np.arange(U)
    pi = np.stack([(a * x + cc) % U for a, cc in ((1, 0), (5, 3), (11, 7), (13, 1))]).astype(np.int64)
    ref = b3.Collection3(off, tids, m, r_min=4, pi=pi)
    assert ref.failures()
    pit = torch.as_tensor(pi.astype(np.int32)).cuda()
    c = _c3(off, tids, m, r_min=4, pi_table=pit, serial=True)
    for i in range(len(off) - 1):
        np.testing.assert_array_equal(c.export_entries(i), ref.bytes[i])
    tri = _all_triples(len(off) - 1)
    got = c.triple_supports(tri, threshold=0).cpu().numpy().astype(np.uint32)
    np.testing.assert_array_equal(got[:, :3], tri.astype(np.uint32))
    np.testing.assert_array_equal(got[:, 3], oracle.triples_list(off, tids, tri[:, 0], tri[:, 1], tri[:, 2]))
    conc = _c3(off, tids, m, r_min=4, pi_table=pit)  # concurrent build under the same colliding π
    got = conc.triple_supports(tri, threshold=0).cpu().numpy().astype(np.uint32)
    np.testing.assert_array_equal(got[:, 3], oracle.triples_list(off, tids, tri[:, 0], tri[:, 1], tri[:, 2]))


def _check_layout(c, off, tids, m, seed, r_min=128):
    s3, U = b3.derive_params3(m)
    P = b3.pi_table4(seed, s3)
    fails = {}
    for it, t in c.failures().tolist():
        fails.setdefault(it, set()).add(t)
    r0 = c.info()["r0"]
    for i in range(len(off) - 1):
        S = tids[off[i]:off[i + 1]].tolist()
        ent = c.export_entries(i)
        r = len(ent) // 4
        assert r == b3.table_range3(len(S), s3, r_min)
        seen = np.zeros(len(ent), bool)
        f = fails.get(i, set())
        assert f <= set(S)
        for x in S:
            if x in f:
                continue
            qs = [b3.h4(t, int(P[t - 1][x]), r, r0) for t in (1, 2, 3, 4)]
            have = [t for t, q in zip((1, 2, 3, 4), qs)
                    if ent[q] != b3.NULL3 and (ent[q] & 0x3F) == (int(P[t - 1][x]) >> s3)]
            assert len(have) == 3, (i, x, have)
            missing = ({1, 2, 3, 4} - set(have)).pop()
            for t in have:
                q = qs[t - 1]
                assert ent[q] == b3.encode_entry3(int(P[t - 1][x]) >> s3, t, missing)
                seen[q] = True
        assert int((ent != b3.NULL3).sum()) == int(seen.sum())


@pytest.mark.parametrize("max_loop", [0, 1])
def test_concurrent_build_invariants_and_supports(max_loop):
    off, tids, m = _instance(11, n=12)
    c = _c3(off, tids, m, seed=4, max_loop=max_loop)
    _check_layout(c, off, tids, m, 4)
    if max_loop:
        assert c.info()["n_failures"] > 0
    tri = _all_triples(len(off) - 1)
    got = c.triple_supports(tri, threshold=0).cpu().numpy().astype(np.uint32)
    np.testing.assert_array_equal(got[:, 3], oracle.triples_list(off, tids, tri[:, 0], tri[:, 1], tri[:, 2]))
    for thr in (1, 50):
        ref = oracle.triples_horizontal(off, tids, m, threshold=thr)
        np.testing.assert_array_equal(c.triple_supports(tri, threshold=thr).cpu().numpy().astype(np.uint32), ref)


def test_big_tables_and_wide_width_mix():
    """Tables from r = 128 to 2^16 in one collection (many chunks per item, long wrap-around)."""
    rng = np.random.default_rng(3)
    m = 200_000
    base = rng.choice(m, size=40000, replace=False)
    rows = []
    for size in (30, 300, 3000, 30000, 30000, 12000, 700):
        rows.append(np.unique(np.concatenate([rng.choice(base, size=size // 2, replace=False),
                                              rng.choice(m, size=size - size // 2)])).astype(np.int32))
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows)
    for max_loop in (0, 1):
        c = _c3(off, tids, m, seed=2, max_loop=max_loop)
        _check_layout(c, off, tids, m, 2)
        tri = _all_triples(len(rows))
        got = c.triple_supports(tri, threshold=0).cpu().numpy().astype(np.uint32)
        np.testing.assert_array_equal(got[:, 3], oracle.triples_list(off, tids, tri[:, 0], tri[:, 1], tri[:, 2]))


def test_candidate_triples_equal_brute_join():
    from paper_1102_1003_b200 import candidate_triples

    rng = np.random.default_rng(8)
    n = 60
    P = sorted({tuple(sorted(rng.choice(n, size=2, replace=False).tolist())) for _ in range(700)})
    pairs = np.array([(i, j, 1) for i, j in P], np.int32)
    got = candidate_triples(torch.as_tensor(pairs).cuda(), n).cpu().numpy()
    S = set(P)
    ref = [(i, j, k) for i, j, k in itertools.combinations(range(n), 3) if (i, j) in S and (i, k) in S and (j, k) in S]
    np.testing.assert_array_equal(got, np.array(ref, np.int32).reshape(-1, 3))
    empty = candidate_triples(torch.zeros((0, 3), dtype=torch.int32).cuda(), n)
    assert empty.shape[0] == 0


def _mine(off, tids, m, thr):
    from paper_1102_1003_b200 import mine_triples

    q, info = mine_triples(torch.as_tensor(off).cuda(), torch.as_tensor(tids).cuda(), m, thr, seed=1)
    return q.cpu().numpy().astype(np.uint32), info


def test_mine_triples_c1_low_threshold():
    w = make_config("C1")
    got, info = _mine(w.offsets, w.tids, w.m, 2)
    ref = oracle.triples_horizontal(w.offsets, w.tids, w.m, threshold=2)
    assert ref.shape[0] > 100
    np.testing.assert_array_equal(got, ref)


def test_mine_triples_c3_quest_official_threshold():
    w = make_config("C3")
    got, info = _mine(w.offsets, w.tids, w.m, w.threshold)
    ref = oracle.triples_horizontal(w.offsets, w.tids, w.m, threshold=w.threshold)
    assert ref.shape[0] > 100 and info["candidates"] >= ref.shape[0]
    np.testing.assert_array_equal(got, ref)


def test_mine_triples_planted():
    """Uniform noise plus planted frequent triples (shared tidlist chunks)."""
    m = 50_000
    off, tids = uniform(400, m, 0.01, 21)
    rows = [tids[off[i]:off[i + 1]] for i in range(400)]
    rng = np.random.default_rng(0)
    for g in range(30):
        common = rng.choice(m, size=int(rng.integers(20, 200)), replace=False)
        for i in rng.choice(400, size=3, replace=False):
            rows[i] = np.union1d(rows[i], common).astype(np.int32)
    off = np.zeros(401, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    tids = np.concatenate(rows)
    got, info = _mine(off, tids, m, 20)
    ref = oracle.triples_horizontal(off, tids, m, threshold=20)
    assert ref.shape[0] >= 25
    np.testing.assert_array_equal(got, ref)


# "" = the default grouped kernel (hoisted parameters, 4 candidates per CTA; r_0 >= 1024); "0" = warp
# per candidate; "h0" = the grouped kernel with shared-memory parameters; "h2" / "h6" / "h8" = other
# candidates-per-CTA counts of the hoisted kernel
@pytest.mark.parametrize("grouped", ["", "0", "h0", "h2", "h6", "h8"])
def test_triple_kernels_any_candidate_order(grouped, monkeypatch):
    """The grouped kernels reuse B_i and B_j across a run of candidates sharing (i, j); they must be
    exact for any candidate order (runs split anywhere, CTAs of any size), with and without
    failures, and agree with the one-warp-per-candidate kernel."""
    if grouped.startswith("h"):
        monkeypatch.setenv("BATMAP_K3_HOIST", grouped[1:])
    elif grouped:
        monkeypatch.setenv("BATMAP_K3_GROUPED", grouped)
    off, tids, m = _instance(21, n=14)
    rng = np.random.default_rng(5)
    tri = _all_triples(len(off) - 1)
    for max_loop in (0, 1):
        c = _c3(off, tids, m, seed=6, max_loop=max_loop, r_min=1024)  # r_0 >= 1024: the grouped kernel's range
        ref = oracle.triples_list(off, tids, tri[:, 0], tri[:, 1], tri[:, 2])
        for order in (np.arange(len(tri)), rng.permutation(len(tri))):
            got = c.triple_supports(np.ascontiguousarray(tri[order]), threshold=0).cpu().numpy().astype(np.uint32)
            np.testing.assert_array_equal(got[:, :3], tri.astype(np.uint32))
            np.testing.assert_array_equal(got[:, 3], ref)
